python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dpkfac.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "asym or inception or kl_clip or stale or default" > gpurun_out/gputest_r2e.log 2>&1; echo rc=$? >> gpurun_out/gputest_r2e.log
python bench.py --model inception_v4 --no-cpu-baseline > gpurun_out/bench_incv4_r2e.json 2> gpurun_out/bench_incv4_r2e.err
python bench.py --model densenet201 --no-cpu-baseline > gpurun_out/bench_dn201_r2e.json 2> gpurun_out/bench_dn201_r2e.err
tail -5 gpurun_out/gputest_r2e.log; head -c 1200 gpurun_out/bench_incv4_r2e.json; tail -3 gpurun_out/bench_incv4_r2e.err; echo; head -c 600 gpurun_out/bench_dn201_r2e.json
