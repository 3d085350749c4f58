python scripts/spd_bench.py
python scripts/prof_step.py --warmup 3 --profiled 3
DPK_CG2=0 python scripts/prof_step.py --warmup 3 --profiled 3
python scripts/kbench.py 2>&1 | head -12
