python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dpkfac.py tests/test_gpu_fullsize.py tests/test_gpu_golden.py -m gpu -q -p no:cacheprovider > gpurun_out/gputest_r2y.log 2>&1; echo rc=$? >> gpurun_out/gputest_r2y.log; tail -3 gpurun_out/gputest_r2y.log
python scripts/taps_one.py 2>&1 | cut -c1-160
for sp in 1 0; do DPK_SYRK_SPLIT=$sp python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b_r2y.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b_r2y.json'));print('split=$sp', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"; done
