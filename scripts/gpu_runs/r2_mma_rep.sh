python scripts/unit_trace.py f16 8192 2>/dev/null | head -3
DPK_LIB_PATH=$PWD/exp_so/libdpkfac_r2.so python scripts/unit_trace.py f16 8192 2>/dev/null | head -3
python scripts/unit_trace.py tf32 8192 2>/dev/null | head -3
DPK_LIB_PATH=$PWD/exp_so/libdpkfac_r2.so python scripts/unit_trace.py tf32 8192 2>/dev/null | head -3
