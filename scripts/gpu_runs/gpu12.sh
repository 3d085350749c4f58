python scripts/factor_breakdown.py 2>&1 | head -14
timeout 900 python -m pytest tests -q -m gpu --tb=short 2>&1 | tail -8
python scripts/prof_step.py --profiled 3 2>&1 | tail -1
python scripts/kbench.py 2>&1 | grep -E "rows_k |im2col"
