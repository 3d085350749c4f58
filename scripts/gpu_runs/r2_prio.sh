for pr in "-2,-1" "-2,0" "-1,0" "-2,-2"; do for m in resnet50 densenet201 inception_v4; do DPK_SIDE_PRIO=$pr python bench.py --model $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('prio $pr $m', round(d['ms_per_step'],3))"; done; done
