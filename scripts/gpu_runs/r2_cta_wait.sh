python scripts/unit_trace.py f16 8192 | head -4
python scripts/unit_trace.py tf32 8192 | head -4
python scripts/unit_trace.py syrk16 256 401408 | head -3
python scripts/f16_peak.py
