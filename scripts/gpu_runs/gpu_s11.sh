for n in 4608 2304 2048 1152 576 512 256; do echo "n=$n"; SPD_ONLY=$n python scripts/spd_bench.py | head -1; done
DPK_SPD_TRACE=1 SPD_ONLY=4608 python scripts/spd_bench.py > gpurun_out/spd_trace4608b.log 2>&1
tail -3 gpurun_out/spd_trace4608b.log
