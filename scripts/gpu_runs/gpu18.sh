DPK_DEBUG_TS=1 python scripts/ts_small.py
python scripts/small_gemm.py
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python scripts/prof_step.py --warmup 3 --profiled 3
