# round-1 (session 3) artifacts: bench line N=1, reference arm, timed-step launch list, ncu captures
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01c_final.json 2> gpurun_out/bench_r01c.err; echo bench=$?
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r01c_final.json 2>> gpurun_out/bench_r01c.err; echo ref=$?
timeout 400 python bench.py --steps 5 --warmup 3 --inv-type eigen --no-cpu-baseline > gpurun_out/bench_r01c_final_eigen.json 2>> gpurun_out/bench_r01c.err; echo eigen=$?
DPK_PROFILE_TIMED=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c_final_launches_timed_step.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:segment_kernel -s 1 -c 1 -o gpurun_out/prof_segment python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo rows=$?
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:tc_gemm_kernel<1, 1, 2>" -s 2 -c 1 -o gpurun_out/prof_syrk python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo syrk=$?
python scripts/ncu_summary.py gpurun_out/r01c_final_ncu_summary.json segment_pack=gpurun_out/prof_segment.ncu-rep syrk_factors=gpurun_out/prof_syrk.ncu-rep 2>&1 | tail -2
cat gpurun_out/bench_r01c_final.json gpurun_out/bench_ref_r01c_final.json gpurun_out/bench_r01c_final_eigen.json
