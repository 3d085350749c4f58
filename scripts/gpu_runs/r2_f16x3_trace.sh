for dt in 3xtf32 3xf16; do for n in 8192 2304; do timeout 300 python scripts/unit_trace.py $dt $n 2>/dev/null | head -3; done; done
DPK_CG2=0 timeout 300 python scripts/unit_trace.py 3xf16 2304 2>/dev/null | head -3
DPK_CG2=0 timeout 300 python scripts/unit_trace.py 3xtf32 2304 2>/dev/null | head -3
