python scripts/leaf_one.py 128 3 && ncu --set full --clock-control none --import-source on -k regex:spd_leaf -s 3 -c 1 -o gpurun_out/prof_leaf2 python scripts/leaf_one.py 128 3 > gpurun_out/ncu26.log 2>&1
echo rc=$?
