set -x
python scripts/implicit_vs_f16.py 20
DPK_TAPS=0 python scripts/implicit_vs_f16.py 20
