timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
TMO=200 timeout 300 python scripts/e2e_probe.py 2>&1 | tail -8
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench9.json 2> gpurun_out/bench9.err; echo bench=$?
cat gpurun_out/bench9.json
