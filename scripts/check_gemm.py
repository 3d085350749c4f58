"""Correctness sweep of the engine's operand paths (TMA and manual) vs torch fp64."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import _lib as L, ops

torch.manual_seed(0)
dev = torch.device("cuda", 0)
bad = 0
for (m, n, k) in [(128, 128, 32), (130, 70, 45), (512, 784, 300), (256, 256, 1000), (1000, 2048, 64)]:
    a = torch.randn(m, k, device=dev); b = torch.randn(n, k, device=dev)
    at, bt = a.t().contiguous(), b.t().contiguous()
    ref = (a.double() @ b.double().t())
    for an, aop in [("rk", ops.operand_rows_k(a)), ("rmn", ops.operand_rows_mn(at))]:
        for bn, bop in [("rk", ops.operand_rows_k(b)), ("rmn", ops.operand_rows_mn(bt))]:
            for prec in ["tf32", "tf32-trunc", "3xtf32"]:
                out = torch.full((m, n), float("nan"), device=dev)
                j = L.GemmJob(); j.a, j.b = aop, bop; j.out, j.ldo = out.data_ptr(), n; j.alpha = 1.0
                ops.gemm([j], prec); torch.cuda.synchronize()
                err = float((out.double() - ref).norm() / ref.norm())
                tol = 2e-5 if prec == "3xtf32" else 2e-3
                flag = "" if err <= tol else "  <-- BAD"
                bad += bool(flag)
                print(f"m={m} n={n} k={k} a={an} b={bn} {prec:10s} err={err:.2e}{flag}")
# SYRK slab path
for (c, h) in [(64, 56), (256, 14), (128, 28)]:
    x = torch.relu(torch.randn(8, c, h, h, device=dev))
    op = ops.operand_im2col(x, (1, 1), (1, 1), (0, 0), (1, 1))
    out = torch.empty(c, c, device=dev)
    ops.syrk_ema([ops.factor_job(op, out, 1.0 / op.cols, 0.0)], "tf32"); torch.cuda.synchronize()
    X = x.permute(1, 0, 2, 3).reshape(c, -1).double()
    ref = X @ X.t() / X.shape[1]
    err = float((out.double() - ref).norm() / ref.norm())
    bad += err > 2e-3
    print(f"slab c={c} h={h} err={err:.2e}")
print("BAD", bad)
# rounding check: positive data exposes truncation bias (~7e-4) vs round-to-nearest (~1e-5)
x = torch.relu(torch.randn(512, 8192, device=dev)) + 0.1
ref = x.double() @ x.double().t() / x.shape[1]
for prec in ["tf32", "tf32-trunc", "3xtf32"]:
    for path, op in [("tma rows_k", ops.operand_rows_k(x)), ("tma rows_mn", ops.operand_rows_mn(x.t().contiguous()))]:
        out = torch.empty(512, 512, device=dev)
        ops.syrk_ema([ops.factor_job(op, out, 1.0 / x.shape[1], 0.0)], prec); torch.cuda.synchronize()
        print(f"rounding {prec:10s} {path:12s} err={float((out.double() - ref).norm() / ref.norm()):.2e}")
