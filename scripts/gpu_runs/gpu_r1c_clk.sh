timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bclk.json 2>gpurun_out/bclk.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bclk.json')); print(round(d['ms_per_step'],3), d['clocks'])"
tail -2 gpurun_out/bclk.err
