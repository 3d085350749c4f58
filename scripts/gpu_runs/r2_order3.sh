run() { python bench.py --steps 20 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), 'e2e', round(d['e2e']['ms_per_iter'],3))"; }
run --factor-order 0
run --factor-order 3
run --factor-order 3 --side-cap 96
run --factor-order 3 --side-cap 128
run --factor-order 0
run --factor-order 3 --model inception_v4
run --factor-order 0 --model inception_v4
