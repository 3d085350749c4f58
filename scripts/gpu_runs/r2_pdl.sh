for v in 0 1; do echo PDL=$v; DPK_PDL=$v SPD_ONLY=4608 python scripts/inv_factor_one.py 10; DPK_PDL=$v python scripts/inv_factor_one.py 10; done
for v in 0 1 0 1; do DPK_PDL=$v python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('PDL=$v', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"; done
