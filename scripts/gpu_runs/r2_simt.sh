set -x
mkdir -p gpurun_out/simt
for cfg in "SPD_ONLY=4608 SPD_COUNT=1" "SPD_ONLY=4608" ""; do
  echo "$cfg: $(env $cfg python scripts/inv_factor_one.py 20 2>&1 | tail -1)" >> gpurun_out/simt/inv.txt
done
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or spd or factored or non_spd or damped or precondition" > gpurun_out/simt/tests.txt 2>&1
tail -3 gpurun_out/simt/tests.txt
DPK_SPD_TRACE=1 SPD_ONLY=4608 SPD_COUNT=1 python scripts/inv_factor_one.py 1 > gpurun_out/simt/trace1.txt 2>&1
python bench.py > gpurun_out/simt/bench.json 2> gpurun_out/simt/bench.err
cat gpurun_out/simt/inv.txt
python - <<'P'
import json
d = json.loads(open("gpurun_out/simt/bench.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d.get("stages_ms"), d["e2e"]["value"], d["clocks"])
P
