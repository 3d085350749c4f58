python scripts/small_gemm.py
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python scripts/prof_step.py --warmup 3 --profiled 3
