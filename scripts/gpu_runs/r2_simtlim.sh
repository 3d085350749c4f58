mkdir -p gpurun_out/simtlim
for v in 5e7 1e8 2e8 2.5e7; do
  echo "SIMT=$v chain1: $(DPK_SIMT_FMA=$v SPD_ONLY=4608 SPD_COUNT=1 python scripts/inv_factor_one.py 20 2>&1 | tail -1)" >> gpurun_out/simtlim/out.txt
  echo "SIMT=$v all: $(DPK_SIMT_FMA=$v python scripts/inv_factor_one.py 20 2>&1 | tail -1)" >> gpurun_out/simtlim/out.txt
  DPK_SIMT_FMA=$v python bench.py --no-cpu-baseline --no-e2e > gpurun_out/simtlim/b_$v.json 2>/dev/null
  echo "SIMT=$v bench: $(python -c "import json;d=json.load(open('gpurun_out/simtlim/b_$v.json'));print(round(d['ms_per_step'],3), d['stages_ms'])")" >> gpurun_out/simtlim/out.txt
done
DPK_SIMT_FMA=5e7 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/simtlim/b_5e7_again.json 2>/dev/null
echo "SIMT=5e7 again: $(python -c "import json;d=json.load(open('gpurun_out/simtlim/b_5e7_again.json'));print(round(d['ms_per_step'],3))")" >> gpurun_out/simtlim/out.txt
cat gpurun_out/simtlim/out.txt
