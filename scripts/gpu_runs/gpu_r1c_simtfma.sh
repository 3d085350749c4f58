for v in 1.5e8 3e8 6e8 1.2e9; do
echo "== DPK_SIMT_FMA=$v"
DPK_SIMT_FMA=$v SPD_ONLY=4608 timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
DPK_SIMT_FMA=$v SPD_ONLY=2304 timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
DPK_SIMT_FMA=$v timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
DPK_SIMT_FMA=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bsf.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bsf.json')); print('bench', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
