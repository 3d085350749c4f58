SPD_ONLY=4608 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/inv4608.csv python scripts/inv_one.py 1 > /dev/null 2>&1
SPD_ONLY=4608 DPK_SPD_TRACE=1 python scripts/spd_bench.py > gpurun_out/tr4608c.log 2>&1
