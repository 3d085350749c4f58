python scripts/one_small.py 128 && ncu --set full --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/prof_small python scripts/one_small.py 128 > gpurun_out/ncu16.log 2>&1
echo rc=$?
