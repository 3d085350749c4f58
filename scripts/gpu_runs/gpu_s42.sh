python -m pytest tests -m gpu -x -q -k "spd or factored or inverse" 2>&1 | tail -2
DPK_LEAF_W=8 python scripts/leaf_prof.py; DPK_LEAF_W=4 python scripts/leaf_prof.py
python scripts/leaf_tri.py 3
SPD_ONLY=4608 python scripts/inv_factor_one.py
DPK_LEAF_W=4 SPD_ONLY=4608 python scripts/inv_factor_one.py
