timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "3xf16" 2>&1 | tail -2
for n in 8192 4608 2304; do for dt in 3xtf32 3xf16; do timeout 300 python scripts/unit_trace.py $dt $n 2>/dev/null | head -3; done; done
