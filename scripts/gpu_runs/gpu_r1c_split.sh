timeout 600 python -m pytest tests -m gpu -x -q -k "spd or inverse or factored or resume" 2>&1 | tail -2
for v in 1 0; do
echo "DPK_SPLIT64=$v"
DPK_SPLIT64=$v SPD_ONLY=4608 timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
DPK_SPLIT64=$v SPD_ONLY=2304 timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
DPK_SPLIT64=$v timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
DPK_SPLIT64=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bsplit_$v.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bsplit_$v.json')); print('bench', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
