python scripts/unit_trace.py syrk16 256 401408 | head -6
python scripts/unit_trace.py syrk16 512 200704 | head -8
python scripts/unit_trace.py syrk16 1024 100352 | head -8
