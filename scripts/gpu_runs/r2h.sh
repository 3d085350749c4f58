# SPD chain trace (ResNet-50 factor set, 4608 only and all) + e2e early-launch variants
SPD_ONLY=4608 DPK_SPD_TRACE=1 python scripts/spd_bench.py > gpurun_out/spd_trace_4608.log 2>&1
DPK_SPD_TRACE=1 python scripts/spd_bench.py > gpurun_out/spd_trace_all.log 2>&1
SPD_ONLY=4608 python scripts/inv_factor_one.py 20 > gpurun_out/inv_4608.log 2>&1
python scripts/inv_factor_one.py 20 > gpurun_out/inv_all.log 2>&1
for v in "" "--early" "--early --early-priority low"; do
  python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 30 $v > gpurun_out/e2e_var.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e2e_var.json'));print('$v', round(d['ms_per_step'],3), round(d['e2e']['ms_per_iter'],3))"
done
tail -3 gpurun_out/spd_trace_4608.log; cat gpurun_out/inv_4608.log gpurun_out/inv_all.log
