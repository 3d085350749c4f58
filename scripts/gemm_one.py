"""One engine GEMM shape, repeated (for ncu captures):  gemm_one.py M N K [prec] [a_layout b_layout] [reps]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import _lib as L, ops
if os.environ.get("DPK_LIB"):
    L.load(os.environ["DPK_LIB"])

m, n, k = (int(v) for v in sys.argv[1:4])
prec = sys.argv[4] if len(sys.argv) > 4 else "tf32"
la = sys.argv[5] if len(sys.argv) > 5 else "k"
lb = sys.argv[6] if len(sys.argv) > 6 else "k"
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 5
dev = torch.device("cuda", 0)
def opnd(rows, lay):
    if lay == "k":
        t = torch.randn(rows, k, device=dev); return t, ops.operand_rows_k(t)
    t = torch.randn(k, rows, device=dev); return t, ops.operand_rows_mn(t)
ta, a = opnd(m, la)
tb, b = opnd(n, lb)
o = torch.empty(m, n, device=dev)
j = L.GemmJob(); j.a, j.b = a, b; j.out, j.ldo = o.data_ptr(), n; j.alpha = 1.0
ops.gemm([j], prec); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps): ops.gemm([j], prec)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
print(f"M={m} N={n} K={k} {prec} {la}{lb}: {ms:.3f} ms {2.0*m*n*k/ms/1e9:.1f} TF/s")
