for ch in "64 56" "128 28" "256 14" "512 7"; do python scripts/im2col16_one.py $ch 20; done
ncu --set full --import-source on --clock-control none -k regex:im2col_k16_tiled -c 1 -o gpurun_out/ncu_im2col16 python scripts/im2col16_one.py 64 56 1 > gpurun_out/ncu_im2col16.log 2>&1
ncu -i gpurun_out/ncu_im2col16.ncu-rep --page details --csv > gpurun_out/ncu_im2col16_details.csv 2>/dev/null
grep -E "Duration|Memory Throughput|DRAM Throughput|Compute \(SM\) Throughput|Achieved Occupancy|Issue Slots Busy|Warp Cycles Per Issued|L1/TEX Hit|Registers Per|Theoretical Occupancy" gpurun_out/ncu_im2col16_details.csv | head -20
