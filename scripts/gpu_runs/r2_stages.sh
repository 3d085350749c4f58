python scripts/f16_peak.py 2>&1 | head -2
for st in 3 4; do echo "STAGES1=$st"; DPK_LIB_PATH=$PWD/exp_so/libdpkfac_s$st.so python scripts/f16_peak.py 2>&1 | head -2; done
