for v in 1.5e8 5e7 2e7 0 1.5e8; do echo SIMT_FMA=$v; DPK_SIMT_FMA=$v SPD_ONLY=4608 python scripts/inv_factor_one.py 10; DPK_SIMT_FMA=$v python scripts/inv_factor_one.py 10; DPK_SIMT_FMA=$v python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('step', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"; done
