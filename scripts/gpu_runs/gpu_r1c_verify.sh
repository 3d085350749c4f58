timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench_default.json')); print(round(d['ms_per_step'],3), round(d['value']), d['e2e']['ms_per_iter'], d['cpu_baseline']['value'], d['clocks'])"
