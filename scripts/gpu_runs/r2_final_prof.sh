# Profiles at HEAD (1 GPU): launch list of one timed step, ncu --set full of the top kernels, stage traffic
set -u
mkdir -p gpurun_out/fp
DPK_PROFILE_TIMED=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/fp/launches_timed_step.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fp/ncu_launch.log 2>&1; echo "launch list rc=$?"
K='--set full --import-source on --clock-control none --profile-from-start off --nvtx --kernel-name-base demangled'
ncu $K --nvtx-include "factors/" -k 'regex:tc_gemm_kernel<\(int\)1, \(bool\)1, \(int\)2,' -c 1 -o gpurun_out/fp/ncu_factor_syrk_pairs python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/fp/ncu1.log 2>&1; echo "syrk rc=$?"
ncu $K --nvtx-include "inversion/" -k 'regex:tc_gemm_kernel<\(int\)3, \(bool\)0, \(int\)2,' -c 1 -o gpurun_out/fp/ncu_spd_round python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/fp/ncu2.log 2>&1; echo "spd rc=$?"
ncu $K --nvtx-include "inversion/" -k 'regex:spd_leaf_kernel' -c 1 -o gpurun_out/fp/ncu_leaf python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/fp/ncu3.log 2>&1; echo "leaf rc=$?"
ncu $K --nvtx-include "precondition/" -k 'regex:tc_gemm_kernel<\(int\)3, \(bool\)0, \(int\)2,' -c 1 -o gpurun_out/fp/ncu_precond python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/fp/ncu4.log 2>&1; echo "precond rc=$?"
ncu $K --nvtx-include "factors/" -k 'regex:im2col_k16_tiled' -c 1 -o gpurun_out/fp/ncu_im2col python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/fp/ncu5.log 2>&1; echo "im2col rc=$?"
bash scripts/stage_traffic.sh resnet50 inverse > gpurun_out/fp/stage_traffic.log 2>&1; cat gpurun_out/fp/stage_traffic.log
mv gpurun_out/stage_traffic_*.csv gpurun_out/fp/ 2>/dev/null
ls gpurun_out/fp
