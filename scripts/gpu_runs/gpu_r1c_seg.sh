timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bseg.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bseg.json')); print('bench', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()}, 'e2e', round(d['e2e']['ms_per_iter'],2))"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:segment_kernel -s 2 -c 2 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | grep segment | cut -c1-300
