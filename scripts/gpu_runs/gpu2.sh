timeout 900 python -m pytest tests/test_gpu_kernels.py -q --tb=line -rf 2>&1 | tail -25
timeout 900 python -m pytest tests/test_gpu_dpkfac.py -q --tb=short -rf 2>&1 | tail -60
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
