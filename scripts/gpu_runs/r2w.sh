python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -x -k "f16 or asym or prescale" > gpurun_out/gputest_r2w.log 2>&1; echo rc=$? >> gpurun_out/gputest_r2w.log; tail -2 gpurun_out/gputest_r2w.log
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b_r2w.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b_r2w.json'));print(round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"
bash scripts/stage_traffic.sh resnet50 inverse > gpurun_out/stage_traffic.log 2>&1; cat gpurun_out/stage_traffic.log
