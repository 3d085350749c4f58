timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "tapmajor or taps" 2>&1 | tail -2
for m in materialize auto; do
timeout 120 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --im2col $m > gpurun_out/btaps_$m.json 2>/dev/null; echo $m rc=$?
python -c "import json; d=json.load(open('gpurun_out/btaps_$m.json')); print('$m', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
DPK_DYN=0 timeout 120 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --im2col auto > gpurun_out/btaps_nodyn.json 2>/dev/null; echo nodyn rc=$?
python -c "import json; d=json.load(open('gpurun_out/btaps_nodyn.json')); print('auto nodyn', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
