timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "spd or inverse or factor_inv or precondition_factored" 2>&1 | tail -3
for v in 0 1; do echo LEAF_MMA=$v; DPK_LEAF_MMA=$v SPD_ONLY=4608 python scripts/inv_factor_one.py 10; DPK_LEAF_MMA=$v python scripts/inv_factor_one.py 10; done
