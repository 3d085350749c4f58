timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 8 -c 1 -o gpurun_out/prof_pre3x python scripts/precond_one.py 1 > /dev/null 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_pre3x.ncu-rep --page source --csv --print-source sass > gpurun_out/pre3x_source.csv 2>&1; echo src=$?
ncu -i gpurun_out/prof_pre3x.ncu-rep --page details --csv > gpurun_out/pre3x_details.csv 2>&1; echo det=$?
ls -la gpurun_out/pre3x_source.csv gpurun_out/pre3x_details.csv
