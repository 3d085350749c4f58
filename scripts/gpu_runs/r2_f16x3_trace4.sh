timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "3xf16 or gemm_all or precondition_factored" 2>&1 | tail -2
for n in 8192 2304; do for dt in 3xtf32 3xf16; do timeout 300 python scripts/unit_trace.py $dt $n 2>/dev/null | head -3; done; done
for dt in 3xtf32 3xf16; do DPK_CG2=0 timeout 300 python scripts/unit_trace.py $dt 2304 2>/dev/null | head -3; done
for t in -1 2e9 5e8; do echo F16_MIN=$t; DPK_SPD_F16_MIN=$t SPD_ONLY=4608 python scripts/inv_factor_one.py 10; DPK_SPD_F16_MIN=$t python scripts/inv_factor_one.py 10; done
