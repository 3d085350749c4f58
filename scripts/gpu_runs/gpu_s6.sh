DPK_DEBUG_TS=1 python scripts/ts_group.py
python scripts/ts_group.py
