timeout 120 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-overlap > gpurun_out/b8a.json 2>/dev/null; echo nooverlap=$?
timeout 120 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b8b.json 2>/dev/null; echo overlap=$?
DPK_DYN=0 timeout 120 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b8c.json 2>/dev/null; echo overlap_nodyn=$?
python - <<'PY'
import json
for f in ("b8a","b8b","b8c"):
    try:
        d=json.load(open(f"gpurun_out/{f}.json")); print(f, d["ms_per_step"], d["ms_per_step_serialized"], d["stages_ms"])
    except Exception as e: print(f, "ERR", e)
PY
