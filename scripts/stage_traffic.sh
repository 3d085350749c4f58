#!/bin/bash
# Whole-stage DRAM traffic of one serialized DP-KFAC step (HEAD), for bench.py's
# roofline.traffic: ncu over the kernels inside each NVTX stage range
# (DPKFAC.nvtx, bench.py --ncu-step), metrics dram__bytes_read/write + duration.
#   bash scripts/stage_traffic.sh [model] [inv_type]   -> gpurun_out/stage_traffic_<stage>.csv
set -u
MODEL=${1:-resnet50}
INV=${2:-inverse}
mkdir -p gpurun_out
for st in factors inversion precondition comm_rs comm_ag; do
  ncu --profile-from-start off --nvtx --nvtx-include "${st}/" --clock-control none \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
      --log-file gpurun_out/stage_traffic_${st}.csv \
      python bench.py --model $MODEL --inv-type $INV --steps 1 --warmup 3 --ncu-step \
      > gpurun_out/stage_traffic_${st}.log 2>&1
  echo "$st rc=$?"
done
