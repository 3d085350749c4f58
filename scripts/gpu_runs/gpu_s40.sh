ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:tc_gemm_kernel<.int.1, .bool.1, .int.2>" -s 1 -c 1 -o gpurun_out/prof_syrk python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-overlap > gpurun_out/ncu_syrk.log 2>&1; echo syrk=$?
tail -3 gpurun_out/ncu_syrk.log
