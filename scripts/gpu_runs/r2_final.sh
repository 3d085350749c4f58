# Round-2 evidence at HEAD (1 GPU): tests, bench lines, reference arm, launch list, ncu captures, stage traffic
set -u
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/gputest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final/gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; echo "ref rc=$?"
for m in resnet32 densenet201 inception_v4; do python bench.py --model $m --no-cpu-baseline > gpurun_out/final/bench_$m.json 2> gpurun_out/final/bench_$m.err; echo "$m rc=$?"; done
python bench.py --inv-type eigen --steps 5 --warmup 3 --e2e-steps 5 --no-cpu-baseline > gpurun_out/final/bench_eigen.json 2> gpurun_out/final/bench_eigen.err; echo "eigen rc=$?"
DPK_PROFILE_TIMED=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final/launches_timed_step.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final/ncu_launch.log 2>&1; echo "launch list rc=$?"
ncu --set full --import-source on --clock-control none --profile-from-start off --nvtx --nvtx-include "factors/" -k regex:tc_gemm_kernel -c 1 -o gpurun_out/final/ncu_factor_syrk python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/final/ncu_full1.log 2>&1; echo "ncu syrk rc=$?"
ncu --set full --import-source on --clock-control none --profile-from-start off --nvtx --nvtx-include "inversion/" -k regex:"tc_gemm_kernel<3, 0, 2>" -c 1 -o gpurun_out/final/ncu_spd_round python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/final/ncu_full2.log 2>&1; echo "ncu spd rc=$?"
ncu --set full --import-source on --clock-control none --profile-from-start off --nvtx --nvtx-include "inversion/" -k regex:spd_leaf_kernel -c 1 -o gpurun_out/final/ncu_leaf python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/final/ncu_full3.log 2>&1; echo "ncu leaf rc=$?"
ncu --set full --import-source on --clock-control none --profile-from-start off --nvtx --nvtx-include "precondition/" -k regex:"tc_gemm_kernel<3, 0, 2>" -c 1 -o gpurun_out/final/ncu_precond python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/final/ncu_full4.log 2>&1; echo "ncu precond rc=$?"
ncu --set full --import-source on --clock-control none --profile-from-start off --nvtx --nvtx-include "factors/" -k regex:im2col_k16_tiled -c 1 -o gpurun_out/final/ncu_im2col python bench.py --steps 1 --warmup 3 --ncu-step > gpurun_out/final/ncu_full5.log 2>&1; echo "ncu im2col rc=$?"
bash scripts/stage_traffic.sh resnet50 inverse > gpurun_out/stage_traffic.log 2>&1; cat gpurun_out/stage_traffic.log
ls -la gpurun_out/final | head -40
