SPD_ONLY=4608 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/chain4608.csv python scripts/inv_factor_one.py 1 > /dev/null 2>&1; echo rc=$?
python scripts/launch_summary.py gpurun_out/chain4608.csv 2>&1 | head -12
