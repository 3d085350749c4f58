DPK_SPD_TRACE=1 python scripts/spd_bench.py > gpurun_out/tr_cg2.log 2>&1
DPK_CG2=0 DPK_SPD_TRACE=1 python scripts/spd_bench.py > gpurun_out/tr_cg1.log 2>&1
