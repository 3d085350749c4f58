mkdir -p gpurun_out/check1
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/check1/gputest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/check1/gputest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/check1/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/check1/smoke.log
python bench.py > gpurun_out/check1/bench.json 2> gpurun_out/check1/bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/check1/bench.json'));print(round(d['ms_per_step'],3), round(d['value'],1), d['e2e'], d['clocks'])"
