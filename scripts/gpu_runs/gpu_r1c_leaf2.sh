DPK_LEAF2=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "spd or factored or non_spd or inverse" 2>&1 | tail -3
DPK_LEAF2=1 timeout 300 python -m pytest tests/test_gpu_dpkfac.py -x -q 2>&1 | tail -2
for v in 0 1; do
DPK_LEAF2=$v SPD_ONLY=4608 timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
DPK_LEAF2=$v timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
DPK_LEAF2=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bl2.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bl2.json')); print('leaf2=$v bench', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
