python scripts/syrk16_pair.py 128 28 && \
ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:tc_gemm_kernel' -s 2 -c 4 \
  -o gpurun_out/ncu_i16 python scripts/syrk16_pair.py 128 28 > gpurun_out/ncu_i16.log 2>&1; tail -3 gpurun_out/ncu_i16.log
