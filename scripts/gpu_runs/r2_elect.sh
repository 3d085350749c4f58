timeout 300 python scripts/unit_trace.py f16 8192 2>/dev/null | head -3
timeout 300 python scripts/unit_trace.py tf32 8192 2>/dev/null | head -3
timeout 300 python scripts/f16_peak.py
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
