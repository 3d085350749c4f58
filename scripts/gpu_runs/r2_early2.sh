run() { python bench.py --steps 20 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_iter'],3))"; }
run
run --early
run --early --early-priority low
run
