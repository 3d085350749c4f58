python scripts/check_gemm.py 2>&1 | grep -E "BAD|slab|rounding" | tail -12
python scripts/kbench.py 2>&1 | grep gemm
timeout 600 python -m pytest tests -q -m gpu --tb=line 2>&1 | tail -8
python scripts/prof_step.py --profiled 3 2>&1 | tail -2
