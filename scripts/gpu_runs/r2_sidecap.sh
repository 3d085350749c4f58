run() { python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"; }
run --side-cap 0
for c in 128 112 96 80 64; do run --side-cap $c; done
run --side-cap 0
