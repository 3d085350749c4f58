DPK_DEBUG_TS=1 python scripts/ts_sym.py
