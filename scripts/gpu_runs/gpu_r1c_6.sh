TAG=base TMO=60 timeout 100 python scripts/early_hang.py 2>&1 | tail -3
TAG=base2 ITERS=60 TMO=80 timeout 100 python scripts/early_hang.py 2>&1 | tail -3
TMO=200 timeout 300 python scripts/e2e_probe.py 2>&1 | tail -12
