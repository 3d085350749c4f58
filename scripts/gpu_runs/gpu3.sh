timeout 900 python -m pytest tests -q -m gpu --tb=short -rf 2>&1 | tail -30
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_r50.err
cat gpurun_out/bench_r50.json
