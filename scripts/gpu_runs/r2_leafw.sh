for w in 4 8; do echo W=$w; DPK_LEAF_W=$w SPD_ONLY=4608 python scripts/inv_factor_one.py 10; DPK_LEAF_W=$w python scripts/inv_factor_one.py 10; done
python scripts/leaf_one.py 2>&1 | tail -3
