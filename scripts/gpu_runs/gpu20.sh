timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
python scripts/prof_step.py --warmup 3 --profiled 3 > gpurun_out/prof20.log 2>&1 && tail -1 gpurun_out/prof20.log && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r50c.csv python scripts/prof_step.py --profiled 1 > gpurun_out/ncu20.log 2>&1
echo rc=$?
