python scripts/leaf_tri.py 148
ncu --set full --import-source on --clock-control none -k regex:spd_leaf_kernel -s 2 -c 1 -o gpurun_out/leafmany python scripts/leaf_tri.py 148 > /dev/null 2>&1
DPK_LEAF_W=4 ncu --set full --import-source on --clock-control none -k regex:spd_leaf_kernel -s 2 -c 1 -o gpurun_out/leafmany4 python scripts/leaf_tri.py 148 > /dev/null 2>&1
