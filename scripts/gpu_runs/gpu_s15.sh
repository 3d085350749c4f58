python scripts/syrk_one.py 4608 1568 k
python scripts/syrk_one.py 4608 1568 k 10 0
python scripts/syrk_one.py 576 100352 k
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/syrk_launches.csv python scripts/syrk_one.py 4608 1568 k 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/syrk4608 python scripts/syrk_one.py 4608 1568 k 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/syrk576 python scripts/syrk_one.py 576 100352 k 2 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
