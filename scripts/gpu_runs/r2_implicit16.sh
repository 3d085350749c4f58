python -m pytest tests/test_gpu_kernels.py -x -q -k "implicit_f16" 2>&1 | tail -15
timeout 300 python scripts/implicit_vs_f16.py 20
