mkdir -p gpurun_out/cap
for c in 112 96 128 104 120 112; do
  python bench.py --side-cap $c --no-cpu-baseline --no-e2e > gpurun_out/cap/b_$c.json 2>/dev/null
  echo "cap=$c $(python -c "import json;d=json.load(open('gpurun_out/cap/b_$c.json'));print(round(d['ms_per_step'],3))")" >> gpurun_out/cap/out.txt
done
cat gpurun_out/cap/out.txt
