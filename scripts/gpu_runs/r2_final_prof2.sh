# the tc_gemm captures: demangled kernel names (template arguments) for the regex
set -u
mkdir -p gpurun_out/fp
K='--set full --import-source on --clock-control none --profile-from-start off --nvtx --kernel-name-base demangled'
ncu $K --nvtx-include "factors/" -k 'regex:tc_gemm_kernel<\(int\)1, \(bool\)1, \(int\)2,' -c 1 -o gpurun_out/fp/ncu_factor_syrk_pairs python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/fp/ncu1.log 2>&1; echo "syrk rc=$?"
ncu $K --nvtx-include "inversion/" -k 'regex:tc_gemm_kernel<\(int\)3, \(bool\)0, \(int\)2,' -c 1 -o gpurun_out/fp/ncu_spd_round python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/fp/ncu2.log 2>&1; echo "spd rc=$?"
ncu $K --nvtx-include "precondition/" -k 'regex:tc_gemm_kernel<\(int\)3, \(bool\)0, \(int\)2,' -c 1 -o gpurun_out/fp/ncu_precond python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/fp/ncu4.log 2>&1; echo "precond rc=$?"
ls gpurun_out/fp
