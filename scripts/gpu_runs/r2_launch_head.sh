mkdir -p gpurun_out/lh
DPK_PROFILE_TIMED=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/lh/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/lh/ncu.log 2>&1; echo rc=$?
python scripts/launch_summary.py gpurun_out/lh/launches.csv | head -25
