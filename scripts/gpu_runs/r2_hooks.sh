mkdir -p gpurun_out/hooks
for m in resnet50 densenet201; do python scripts/e2e_hooks.py $m >> gpurun_out/hooks/out.txt 2>&1; done
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/hooks/gputest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/hooks/gputest.log
python bench.py > gpurun_out/hooks/bench.json 2> gpurun_out/hooks/bench.err
python -c "import json;d=json.load(open('gpurun_out/hooks/bench.json'));print(round(d['ms_per_step'],3), d['e2e'])"
python bench.py --model densenet201 --no-cpu-baseline > gpurun_out/hooks/bench_dn.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/hooks/bench_dn.json'));print(round(d['ms_per_step'],3), d['e2e'])"
cat gpurun_out/hooks/out.txt
