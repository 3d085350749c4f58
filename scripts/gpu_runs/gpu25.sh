python scripts/leaf_one.py 128 3
python scripts/leaf_one.py 64 3
python scripts/leaf_one.py 20 3
python scripts/spd_bench.py
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
