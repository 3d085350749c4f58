SPD_ONLY=4608 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:bool\)0, \(int\)2" -s 4 -c 1 -o gpurun_out/cg2x3 python scripts/inv_factor_one.py 1 > gpurun_out/ncu_cg2.log 2>&1
SPD_ONLY=4608 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:bool\)0, \(int\)1" -s 25 -c 1 -o gpurun_out/cg1x3 python scripts/inv_factor_one.py 1 > gpurun_out/ncu_cg1.log 2>&1
ls gpurun_out/cg*; tail -2 gpurun_out/ncu_cg2.log
