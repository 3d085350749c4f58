set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "tapmajor or taps or im2col" 2>&1 | tail -8
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench=$?
cat gpurun_out/bench2.json; tail -3 gpurun_out/bench2.err
timeout 600 python scripts/factor_breakdown.py > gpurun_out/fb2.log 2>&1; head -30 gpurun_out/fb2.log
timeout 600 python scripts/e2e_probe.py 2>&1 | tail -12
