run() { env "$@" python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"; }
run DPK_NOP=1
run DPK_UNITS_PER_CTA=1
run DPK_UNITS_PER_CTA=2
run DPK_UNITS_PER_CTA=4
run DPK_GRID_CAP=136
run DPK_GRID_CAP=120
run DPK_NOP=1
