python scripts/unit_trace.py f16 8192 | head -14
python scripts/unit_trace.py tf32 8192 | head -14
