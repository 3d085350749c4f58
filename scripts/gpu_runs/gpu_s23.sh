SPD_ONLY=4608 ncu --set full --import-source on --clock-control none -k regex:spd_leaf_kernel -s 40 -c 1 -o gpurun_out/leaf8 python scripts/inv_one.py 2 > /dev/null 2>&1
SPD_ONLY=4608 ncu --set full --import-source on --clock-control none -k regex:simt_gemm -s 200 -c 1 -o gpurun_out/simt python scripts/inv_one.py 2 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
