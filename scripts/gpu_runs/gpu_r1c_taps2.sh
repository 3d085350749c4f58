timeout 300 python scripts/taps_one.py 2>&1 | tail -8
ONLY=0 timeout 300 ncu --set full --clock-control none -k regex:tc_gemm -s 3 -c 1 -o gpurun_out/prof_taps python scripts/taps_one.py > /dev/null 2>&1; echo ncu=$?
ONLY=0 timeout 300 ncu --set full --clock-control none -k regex:tc_gemm -s 4 -c 1 -o gpurun_out/prof_mn3 python scripts/taps_one.py > /dev/null 2>&1; echo ncu=$?
python scripts/ncu_summary.py gpurun_out/taps_vs_mn3.json taps=gpurun_out/prof_taps.ncu-rep mn3=gpurun_out/prof_mn3.ncu-rep > /dev/null 2>&1; cat gpurun_out/taps_vs_mn3.json
