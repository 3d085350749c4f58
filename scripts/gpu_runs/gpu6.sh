python scripts/prof_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r50.csv python scripts/prof_step.py > gpurun_out/ncu_launch.log 2>&1
echo "rc=$?"
python scripts/prof_step.py > gpurun_out/prof_plain2.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -c 1 -o gpurun_out/prof_syrk python scripts/prof_step.py > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
