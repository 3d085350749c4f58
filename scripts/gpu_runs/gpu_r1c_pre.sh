timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --model resnet32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r01c_resnet32.json 2> /dev/null; echo r32=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01c_resnet32.json')); print('resnet32', round(d['ms_per_step'],3), round(d['value']), 'e2e', round(d['e2e']['ms_per_iter'],2))"
timeout 120 python scripts/precond_one.py 10 2>&1 | tail -1
timeout 300 ncu --set full --clock-control none -k regex:tc_gemm -s 8 -c 4 -o gpurun_out/prof_precond python scripts/precond_one.py 1 > /dev/null 2>&1; echo ncu_pre=$?
timeout 300 ncu --set full --clock-control none -k regex:segment_kernel -s 2 -c 2 -o gpurun_out/prof_segment python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu_seg=$?
ncu -i gpurun_out/prof_precond.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size > gpurun_out/precond_ncu.csv 2>&1; cat gpurun_out/precond_ncu.csv | cut -c1-400 | head -8
ncu -i gpurun_out/prof_segment.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/segment_ncu.csv 2>&1; cat gpurun_out/segment_ncu.csv | cut -c1-400 | head -6
