TMO=200 timeout 300 python scripts/e2e_probe.py 2>&1 | tail -60
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench=$?
cat gpurun_out/bench4.json; tail -3 gpurun_out/bench4.err
