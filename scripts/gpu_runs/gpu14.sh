python scripts/factor_breakdown.py 2>&1 | head -14
timeout 900 python -m pytest tests -q -m gpu --tb=line 2>&1 | tail -5
python scripts/prof_step.py --profiled 3 2>&1 | tail -1
