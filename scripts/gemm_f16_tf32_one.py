"""8192^3 engine GEMM, f16 (kind::f16) then tf32 (1-pass), 2 launches each (ncu target)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import _lib as L, ops
N = 8192
for dt in ("f16", "tf32"):
    a = torch.randn(N, N, device="cuda")
    b = torch.randn(N, N, device="cuda")
    c = torch.empty(N, N, device="cuda")
    j = L.GemmJob()
    if dt == "f16":
        a, b = a.half(), b.half()
        j.a, j.b = ops.operand_rows_k_f16(a, N), ops.operand_rows_k_f16(b, N)
    else:
        j.a, j.b = ops.operand_rows_k(a), ops.operand_rows_k(b)
    j.out, j.ldo, j.alpha = c.data_ptr(), N, 1.0
    for _ in range(2):
        ops.gemm([j], "tf32")
    torch.cuda.synchronize()
