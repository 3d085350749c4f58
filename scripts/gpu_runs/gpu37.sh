python scripts/spd_bench.py
DPK_CG2=0 python scripts/spd_bench.py
python scripts/prof_step.py --warmup 3 --profiled 3
DPK_CG2=0 python scripts/prof_step.py --warmup 3 --profiled 3
DPK_SPD_TRACE=1 python scripts/spd_bench.py 2>&1 | grep -E "4608x4608|2304x2304|1152x1152|^total" | tail -8
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
