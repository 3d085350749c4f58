python scripts/kbench.py > gpurun_out/kbench.log 2>&1
python scripts/spd_bench.py > gpurun_out/spd.log 2>&1
DPK_SPD_TRACE=1 python scripts/spd_bench.py > gpurun_out/spd_trace.log 2>&1
DPK_SPD_TRACE=1 SPD_ONLY=4608 python scripts/spd_bench.py > gpurun_out/spd_trace4608.log 2>&1
tail -5 gpurun_out/spd.log
