python scripts/kbench.py 2>&1 | tail -30
timeout 600 python -m pytest tests -q -m gpu -x --tb=short 2>&1 | tail -15
python scripts/prof_step.py --profiled 3 2>&1 | tail -2
