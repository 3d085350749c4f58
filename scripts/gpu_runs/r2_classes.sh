run() { python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"; }
run
run --max-classes 2
run --max-classes 4
run --class-ratio 0.4
run --class-ratio 0.8
run
