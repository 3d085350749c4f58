set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_r2d.log 2>&1; echo rc=$? >> gpurun_out/gputest_r2d.log
python scripts/tf32_peak.py gpurun_out/tf32_peak.json > gpurun_out/tf32_peak.log 2>&1
python bench.py > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_r2d.json 2> gpurun_out/bench_ref_r2d.err
bash scripts/stage_traffic.sh resnet50 inverse > gpurun_out/stage_traffic.log 2>&1
tail -3 gpurun_out/gputest_r2d.log; cat gpurun_out/bench_r2d.json | head -c 3000; echo; head -c 1500 gpurun_out/bench_ref_r2d.json; cat gpurun_out/stage_traffic.log
