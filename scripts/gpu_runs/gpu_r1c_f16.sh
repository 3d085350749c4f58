timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "f16" 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bf16.json 2>gpurun_out/bf16.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bf16.json')); print('bench', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()}, 'e2e', round(d['e2e']['ms_per_iter'],2))"
tail -3 gpurun_out/bf16.err
