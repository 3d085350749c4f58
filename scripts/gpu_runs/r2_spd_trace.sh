SPD_ONLY=4608 python scripts/inv_factor_one.py 10
python scripts/inv_factor_one.py 10
SPD_ONLY=4608 DPK_SPD_TRACE=1 DPK_SPD_GRAPH=0 python scripts/inv_factor_one.py 1 2>&1 | tail -150 > gpurun_out/spd_trace_4608.txt
head -5 gpurun_out/spd_trace_4608.txt; tail -12 gpurun_out/spd_trace_4608.txt
