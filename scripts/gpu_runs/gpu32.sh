python scripts/spd_bench.py
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
DPK_SPD_TRACE=1 python scripts/spd_bench.py > gpurun_out/spd_trace3.log 2>&1
python scripts/prof_step.py --warmup 3 --profiled 3
