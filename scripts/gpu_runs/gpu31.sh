DPK_PROFILE_TIMED=1 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:tc_gemm_kernel<.int.3' -s 201 -c 1 -o gpurun_out/prof_inv_r01 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_inv_r01.log 2>&1
echo inv rc=$?
DPK_PROFILE_TIMED=1 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:tc_gemm_kernel<.int.1' -s 0 -c 1 -o gpurun_out/prof_syrk_r01 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_syrk_r01.log 2>&1
echo syrk rc=$?
