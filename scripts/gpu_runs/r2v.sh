python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -x -k "f16 or asym or prescale" > gpurun_out/gputest_r2v.log 2>&1; echo rc=$? >> gpurun_out/gputest_r2v.log; tail -3 gpurun_out/gputest_r2v.log
for ch in "64 56" "128 28" "256 14" "512 7"; do python scripts/im2col16_one.py $ch 20; done
python scripts/taps_one.py
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b_r2v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b_r2v.json'));print(round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"
ncu --set full --import-source on --clock-control none -k regex:im2col_k16_tiled -c 1 -o gpurun_out/ncu_im2col16_v2 python scripts/im2col16_one.py 64 56 1 > gpurun_out/ncu_im2col16_v2.log 2>&1
ncu -i gpurun_out/ncu_im2col16_v2.ncu-rep --page details --csv > gpurun_out/ncu_im2col16_v2_details.csv 2>/dev/null
grep -E "\"Duration\"|DRAM Throughput|Compute \(SM\) Throughput|Issue Slots Busy|Executed Instructions\"" gpurun_out/ncu_im2col16_v2_details.csv | head -8
