mkdir -p gpurun_out/split
for sm in 64 32 16; do for u in 0 2 3; do
  ev="DPK_SPLIT_MIN=$sm"; [ $u -gt 0 ] && ev="$ev DPK_UNITS_PER_SM=$u"
  for cfg in "SPD_ONLY=4608 SPD_COUNT=1" "SPD_ONLY=4608"; do
    echo "$ev $cfg: $(env $ev $cfg python scripts/inv_factor_one.py 20 2>&1 | tail -1)" >> gpurun_out/split/inv.txt
  done
done; done
cat gpurun_out/split/inv.txt
