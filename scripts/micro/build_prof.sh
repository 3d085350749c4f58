#!/bin/bash
# libdpkfac_prof.so: the library with -DDPK_LEAF_PROF (per-phase leaf cycle counters)
set -e
cd "$(dirname "$0")/../.."
out=scripts/micro/prof_obj; mkdir -p $out
for f in paper_2206_15143_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -diag-suppress 177 -DDPK_LEAF_PROF -c $f -o $out/$(basename $f .cu).o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/micro/libdpkfac_prof.so $out/*.o
rm -rf $out
