python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py -m gpu -q -p no:cacheprovider -k "eig" -x > gpurun_out/gputest_r2i.log 2>&1; echo rc=$? >> gpurun_out/gputest_r2i.log
tail -30 gpurun_out/gputest_r2i.log
SPD_ONLY=4608 timeout 300 python scripts/eig_bench.py 2 2>&1 | tail -3
timeout 600 python scripts/eig_bench.py 2 2>&1 | tail -3
