SPD_ONLY=4608 timeout 120 python scripts/inv_factor_one.py 10 2>&1 | tail -2
SPD_ONLY=4608 DPK_SPD_TRACE=1 timeout 120 python scripts/inv_factor_one.py 1 > gpurun_out/spd_trace_4608.txt 2>&1; tail -3 gpurun_out/spd_trace_4608.txt
timeout 120 python scripts/inv_factor_one.py 10 2>&1 | tail -1
SPD_ONLY=2304 timeout 120 python scripts/inv_factor_one.py 10 2>&1 | tail -1
SPD_ONLY=576 timeout 120 python scripts/inv_factor_one.py 10 2>&1 | tail -1
SPD_ONLY=128 timeout 120 python scripts/inv_factor_one.py 10 2>&1 | tail -1
