timeout 300 python scripts/taps_one.py 2>&1 | tail -6
DPK_TAPS4D=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "tapmajor or taps" 2>&1 | tail -1
DPK_TAPS4D=1 timeout 300 python scripts/taps_one.py 2>&1 | tail -6
