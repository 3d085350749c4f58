DPK_SPD_TRACE=1 python scripts/spd_bench.py > gpurun_out/spd_trace.log 2>&1
echo rc=$?
