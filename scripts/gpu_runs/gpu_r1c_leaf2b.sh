DPK_LEAF2=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "spd or factored or non_spd or inverse" 2>&1 | tail -1
for v in 0 1; do
DPK_LEAF2=$v SPD_ONLY=4608 timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
DPK_LEAF2=$v SPD_ONLY=128 timeout 120 python scripts/inv_factor_one.py 200 2>&1 | tail -1
done
