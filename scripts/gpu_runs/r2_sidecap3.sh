timeout 1500 python -m pytest tests/test_gpu_dpkfac.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('resnet50', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), d['e2e']['ms_per_iter'])"
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --side-cap 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('resnet50 nocap', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), d['e2e']['ms_per_iter'])"
