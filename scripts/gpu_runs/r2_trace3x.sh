timeout 300 python scripts/unit_trace.py 3xtf32 8192 2>/dev/null | head -4
timeout 300 python scripts/unit_trace.py 3xtf32 2304 2>/dev/null | head -4
DPK_CG2=0 timeout 300 python scripts/unit_trace.py 3xtf32 2304 2>/dev/null | head -4
DPK_CG2=0 timeout 300 python scripts/unit_trace.py tf32 4096 2>/dev/null | head -4
