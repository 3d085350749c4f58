timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:prep_kernel -c 3 --csv python scripts/inv_factor_one.py 1 2>/dev/null | grep prep | cut -c1-200
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bprep.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bprep.json')); print('bench', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
