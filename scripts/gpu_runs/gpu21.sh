python scripts/spd_bench.py
DPK_SPD_TRACE=1 python scripts/spd_bench.py 2>&1 | tail -80
