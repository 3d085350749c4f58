python scripts/spd_bench.py
DPK_SPD_TRACE=1 python scripts/spd_bench.py > gpurun_out/spd_trace2.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python scripts/prof_step.py --warmup 3 --profiled 3
