python scripts/im2col_one.py 256 14 && ncu --set full --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/prof_im2col python scripts/im2col_one.py 256 14 > gpurun_out/ncu13.log 2>&1
python scripts/factor_breakdown.py 2>&1 | head -8
python scripts/prof_step.py --profiled 3 2>&1 | tail -1
