python scripts/inv_factor_one.py
SPD_ONLY=4608 python scripts/inv_factor_one.py
SPD_ONLY=2304 python scripts/inv_factor_one.py
SPD_ONLY=4608 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/finv4608.csv python scripts/inv_factor_one.py 1 > /dev/null 2>&1
