python scripts/gemm_probe.py
