set -x
mkdir -p gpurun_out/la2
for la in 1 0; do
  for cfg in "SPD_ONLY=4608 SPD_COUNT=1" "SPD_ONLY=128" ""; do
    echo "LA=$la $cfg: $(env DPK_LEAF_LA=$la $cfg python scripts/inv_factor_one.py 20 2>&1 | tail -1)" >> gpurun_out/la2/inv.txt
  done
done
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "leaf or factored_spd or non_spd" > gpurun_out/la2/tests.txt 2>&1
tail -3 gpurun_out/la2/tests.txt
DPK_SPD_TRACE=1 SPD_ONLY=4608 SPD_COUNT=1 python scripts/inv_factor_one.py 1 > gpurun_out/la2/trace1.txt 2>&1
cat gpurun_out/la2/inv.txt
