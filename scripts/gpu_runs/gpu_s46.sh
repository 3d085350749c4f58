for i in 1 2; do
timeout 120 python scripts/gemm_one.py 8192 8192 8192 tf32
timeout 120 env DPK_LIB=scripts/micro/libdpkfac_old.so python scripts/gemm_one.py 8192 8192 8192 tf32
timeout 120 python scripts/gemm_one.py 4608 4608 4608 tf32
timeout 120 env DPK_LIB=scripts/micro/libdpkfac_old.so python scripts/gemm_one.py 4608 4608 4608 tf32
done
