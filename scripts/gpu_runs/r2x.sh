python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dpkfac.py -m gpu -q -p no:cacheprovider -x -k "f16 or asym or prescale or inception or conv" > gpurun_out/gputest_r2x.log 2>&1; echo rc=$? >> gpurun_out/gputest_r2x.log; tail -2 gpurun_out/gputest_r2x.log
python scripts/im2col16_stem.py
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:im2col_k16_rows -c 1 python scripts/im2col16_stem.py 1 2>&1 | grep -E "gpu__time|dram__bytes"
