run() { python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"; }
for c in 0 96 112 128; do run --side-cap $c; done
for m in densenet201 inception_v4 resnet32; do run --model $m; done
