timeout 300 python scripts/gemm_probe.py; echo probe rc=$?
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
