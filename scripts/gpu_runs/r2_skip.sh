mkdir -p gpurun_out/skip
for v in 1 0; do
  for cfg in "SPD_ONLY=4608 SPD_COUNT=1" "SPD_ONLY=4608" "SPD_ONLY=128" ""; do
    echo "SKIP=$v $cfg: $(env DPK_LEAF_SKIP=$v $cfg python scripts/inv_factor_one.py 20 2>&1 | tail -1)" >> gpurun_out/skip/inv.txt
  done
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -x -k "spd or factored or non_spd or damped or precondition or fullsize or resnet" > gpurun_out/skip/tests.txt 2>&1
tail -2 gpurun_out/skip/tests.txt
python bench.py > gpurun_out/skip/bench.json 2> gpurun_out/skip/bench.err
cat gpurun_out/skip/inv.txt
python -c "import json;d=json.load(open('gpurun_out/skip/bench.json'));print(round(d['ms_per_step'],3), d['stages_ms'], d['e2e']['ms_per_iter'])"
