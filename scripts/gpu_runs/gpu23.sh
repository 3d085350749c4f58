python scripts/small_gemm.py 2>&1 | grep spd
python scripts/spd_bench.py
DPK_SPD_TRACE=1 python scripts/spd_bench.py 2>&1 | tail -12
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
python scripts/prof_step.py --warmup 3 --profiled 3
