set -x
mkdir -p gpurun_out/la
for la in 1 0; do
  for cfg in "SPD_ONLY=4608 SPD_COUNT=1" "SPD_ONLY=4608" "SPD_ONLY=128" ""; do
    echo "LA=$la $cfg: $(env DPK_LEAF_LA=$la $cfg python scripts/inv_factor_one.py 20 2>&1 | tail -1)" >> gpurun_out/la/inv.txt
  done
done
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "spd or factored or non_spd or leaf or damped or precondition" > gpurun_out/la/tests.txt 2>&1
tail -3 gpurun_out/la/tests.txt
python bench.py > gpurun_out/la/bench_la1.json 2> gpurun_out/la/bench_la1.err
DPK_LEAF_LA=0 python bench.py > gpurun_out/la/bench_la0.json 2> gpurun_out/la/bench_la0.err
cat gpurun_out/la/inv.txt
python - <<'P'
import json
for f in ("la1", "la0"):
    d = json.loads(open(f"gpurun_out/la/bench_{f}.json").read().strip().splitlines()[-1])
    print(f, d["ms_per_step"], d.get("stages_ms"), d["e2e"]["value"])
P
