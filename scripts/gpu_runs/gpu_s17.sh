python scripts/syrk_one.py 147 401408 mn
DPK_CG2=0 python scripts/syrk_one.py 147 401408 mn
python scripts/syrk_one.py 576 100352 mn
DPK_CG2=0 python scripts/syrk_one.py 576 100352 mn
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/syrk147.csv python scripts/syrk_one.py 147 401408 mn 2 > /dev/null 2>&1
