TMO=100 timeout 150 python scripts/early_debug.py 2>&1 | tail -40
CHK=sync TMO=100 timeout 150 python scripts/early_debug.py 2>&1 | tail -12
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "tapmajor or taps or im2col" 2>&1 | tail -4
