for s in 8 16 32; do DPK_EIG_STREAMS=$s python bench.py --inv-type eigen --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('streams $s', round(d['ms_per_step'],1), round(d['stages_ms']['inversion'],1))"; done
