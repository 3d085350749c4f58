python scripts/taps_one.py
for m in materialize auto implicit; do python bench.py --im2col $m --no-cpu-baseline --no-e2e > gpurun_out/im2col_$m.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/im2col_$m.json'));print('$m', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"; done
