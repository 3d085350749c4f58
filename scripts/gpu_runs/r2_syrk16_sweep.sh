TAG=default python scripts/syrk16_sweep.py
for u in 1 3 4 6; do TAG=units$u DPK_UNITS_PER_SM=$u python scripts/syrk16_sweep.py; done
for s in 16 32 128; do TAG=splitmin$s DPK_SPLIT_MIN=$s python scripts/syrk16_sweep.py; done
TAG=cg1 DPK_CG2=0 python scripts/syrk16_sweep.py
