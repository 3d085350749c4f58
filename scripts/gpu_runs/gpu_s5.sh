python scripts/gemm_one.py 4608 4608 4608 3xtf32
DPK_ARRIVE_WARP=1 python scripts/gemm_one.py 4608 4608 4608 3xtf32
python scripts/gemm_one.py 8192 8192 8192 3xtf32
DPK_ARRIVE_WARP=1 python scripts/gemm_one.py 8192 8192 8192 3xtf32
python scripts/inv_one.py
DPK_ARRIVE_WARP=1 python scripts/inv_one.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/inv_launches.csv python scripts/inv_one.py 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o gpurun_out/g4608x3 python scripts/gemm_one.py 4608 4608 4608 3xtf32 k k 1 > /dev/null 2>&1
ls gpurun_out
