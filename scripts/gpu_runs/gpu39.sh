python scripts/spd_bench.py
python scripts/prof_step.py --warmup 3 --profiled 3
DPK_SPD_TRACE=1 python scripts/spd_bench.py > gpurun_out/tr_cg2b.log 2>&1
