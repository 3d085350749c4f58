timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dpkfac.py -x -q 2>&1 | tail -2
for v in 0 1; do for m in resnet50 densenet201 inception_v4; do DPK_CHUNK_FORK=$v python bench.py --model $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('fork $v $m', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"; done; done
