# round artifacts: bench line (N=1), reference arm, timed-step launch list, ncu captures of the top kernels
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench_full.err; echo ref=$?
DPK_PROFILE_TIMED=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_timed_step.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches=$?
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:bool\)1, \(int\)2" -s 2 -c 1 -o gpurun_out/prof_syrk python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo syrk=$?
SPD_ONLY=4608 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:bool\)0, \(int\)2" -s 4 -c 1 -o gpurun_out/prof_spd3x python scripts/inv_factor_one.py 1 > /dev/null 2>&1; echo spd=$?
SPD_ONLY=4608 ncu --set full --import-source on --clock-control none -k regex:spd_leaf -s 40 -c 1 -o gpurun_out/prof_leaf python scripts/inv_factor_one.py 1 > /dev/null 2>&1; echo leaf=$?
SPD_ONLY=4608 ncu --set full --import-source on --clock-control none -k regex:simt_gemm -s 150 -c 1 -o gpurun_out/prof_simt python scripts/inv_factor_one.py 1 > /dev/null 2>&1; echo simt=$?
ncu --set full --import-source on --clock-control none -k regex:im2col_vec -s 1 -c 1 -o gpurun_out/prof_im2col python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo im2col=$?
cat gpurun_out/bench_full.json gpurun_out/bench_ref.json
