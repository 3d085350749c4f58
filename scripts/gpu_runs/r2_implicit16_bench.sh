for v in "--im2col materialize" "--im2col implicit16" "--im2col implicit16 DPK_I16_MAXC=64" "--im2col implicit16 DPK_I16_MAXC=128"; do
  set -- $v
  env ${3:-DPK_NOP=1} python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $1 $2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"
done
