python scripts/gemm_one.py 4608 4608 4608 tf32 > gpurun_out/g1.log 2>&1
python scripts/gemm_one.py 8192 8192 8192 tf32 >> gpurun_out/g1.log 2>&1
python scripts/gemm_one.py 8192 8192 8192 3xtf32 >> gpurun_out/g1.log 2>&1
cat gpurun_out/g1.log
ncu --set full --import-source on -k regex:tc_gemm -c 1 -o gpurun_out/g4608 python scripts/gemm_one.py 4608 4608 4608 tf32 k k 1 > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
