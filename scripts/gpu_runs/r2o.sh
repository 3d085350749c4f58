for rel in 2e-7 1e-6 4e-6; do
  for cfg in "128 24 64" "128 24 400" "64 24 32" "256 8 100"; do DPK_JAC_REL=$rel DPK_EIG_SWEEPS=4 python scripts/jac_one.py $cfg; done
done
