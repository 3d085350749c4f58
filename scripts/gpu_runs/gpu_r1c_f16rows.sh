timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "f16" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/f16_one.py 2>&1 | tail -1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bf16r.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bf16r.json')); print('bench', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
