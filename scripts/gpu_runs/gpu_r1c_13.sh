for u in 0 1 2 4 8; do
  DPK_UNITS_PER_CTA=$u timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b13_$u.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/b13_$u.json')); print('upc=$u', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
for c in 132 140; do
  DPK_GRID_CAP=$c timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b13_c$c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/b13_c$c.json')); print('cap=$c', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"
done
