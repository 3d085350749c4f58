python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/leaf_one.py 128 3
DPK_LEAF_W=4 python scripts/leaf_one.py 128 3
SPD_ONLY=4608 python scripts/spd_bench.py 2>/dev/null | head -1
DPK_LEAF_W=4 SPD_ONLY=4608 python scripts/spd_bench.py 2>/dev/null| head -1
python scripts/spd_bench.py 2>/dev/null
