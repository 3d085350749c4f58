python scripts/check_gemm.py 2>&1 | grep -E "BAD|slab" | tail -40
echo "---- no TMA"
DPK_DISABLE_TMA=1 python scripts/check_gemm.py 2>&1 | grep -E "BAD" | tail -5
python scripts/kbench.py 2>&1 | tail -30
