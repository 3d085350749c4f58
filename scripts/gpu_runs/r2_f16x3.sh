timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "3xf16 or precondition_factored" 2>&1 | tail -4
DPK_SPD_F16_MIN=0 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "spd or inverse or factor" 2>&1 | tail -4
for t in -1 2e9 5e8 1e8 0; do echo "F16_MIN=$t"; DPK_SPD_F16_MIN=$t SPD_ONLY=4608 python scripts/inv_factor_one.py 10; DPK_SPD_F16_MIN=$t python scripts/inv_factor_one.py 10; done
