python scripts/prof_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r50b.csv python scripts/prof_step.py > gpurun_out/ncu_launch.log 2>&1
echo rc=$?
