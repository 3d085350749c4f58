mkdir -p gpurun_out/rowo
for v in 1 0; do
  for cfg in "SPD_ONLY=4608 SPD_COUNT=1" "SPD_ONLY=4608" "SPD_ONLY=128" ""; do
    echo "ROWO=$v $cfg: $(env DPK_LEAF_ROWO=$v $cfg python scripts/inv_factor_one.py 20 2>&1 | tail -1)" >> gpurun_out/rowo/inv.txt
  done
done
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "leaf or spd or factored or non_spd or damped or precondition" > gpurun_out/rowo/tests.txt 2>&1
tail -2 gpurun_out/rowo/tests.txt
python bench.py > gpurun_out/rowo/bench.json 2> gpurun_out/rowo/bench.err
cat gpurun_out/rowo/inv.txt
python -c "import json;d=json.load(open('gpurun_out/rowo/bench.json'));print(round(d['ms_per_step'],3), d['stages_ms'], d['e2e']['ms_per_iter'] if 'ms_per_iter' in d['e2e'] else d['e2e'], d['clocks'])"
