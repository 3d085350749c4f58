for cfg in "128 24 64" "128 24 400" "64 24 32" "10 4 3"; do python scripts/jac_one.py $cfg; done
for sw in 4 6; do DPK_EIG_SWEEPS=$sw timeout 600 python scripts/eig_sizes.py; done
