timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/prof_syrk_f16 python scripts/syrk_f16_one.py f16 > /dev/null 2>&1; echo f16=$?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/prof_syrk_f32 python scripts/syrk_f16_one.py f32 > /dev/null 2>&1; echo f32=$?
