timeout 300 python scripts/unit_trace.py f16 8192 2>/dev/null | head -3
timeout 300 python scripts/unit_trace.py tf32 8192 2>/dev/null | head -3
timeout 300 python scripts/f16_peak.py
timeout 300 python scripts/tf32_peak.py 2>&1 | grep -i 'tflops'
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dpkfac.py -x -q 2>&1 | tail -3
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('resnet50', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"
