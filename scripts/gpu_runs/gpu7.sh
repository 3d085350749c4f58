python scripts/prof_step.py --profiled 3 2>&1 | tail -2
timeout 600 python -m pytest tests -q -m gpu -x --tb=line 2>&1 | tail -3
