"""Timeline (DPK_DEBUG_TS=1) of symmetric beta=1 Schur-style GEMMs vs plain ones."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2206_15143_b200 import _lib as L, ops

names = ["start", "setup", "tma_done", "gather_done", "mma_done", "epi_u0", "epi_last", "final_bar", "dealloc",
         "epi_tfull", "epi_ld0", "epi_st0", "st_done", "sts_done", "lds_done", "math_done"]
lib = L.load()


def run(n, k, sym, beta, prec, reps=20):
    a = torch.randn(n, k, device="cuda")
    o = torch.randn(n, n, device="cuda")
    j = L.GemmJob()
    j.a = ops.operand_rows_k(a)
    j.b = ops.operand_rows_k(a)
    j.out, j.ldo = o.data_ptr(), n
    j.alpha = -1.0
    j.beta = beta
    if beta:
        j.cin, j.ldc = o.data_ptr(), n
    j.symmetric = sym
    for _ in range(3):
        ops.gemm([j], prec)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 16)()
    lib.dpk_debug_timestamps(buf)
    t0 = buf[0]
    tl = {names[i]: round((buf[i] - t0) / 1000.0, 2) for i in range(16) if buf[i] >= t0}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ops.gemm([j], prec)
    e1.record()
    torch.cuda.synchronize()
    print(f"n={n} k={k} sym={sym} beta={beta} {prec}: {e0.elapsed_time(e1) / reps * 1000:.1f} us/call  {tl}")


for sym, beta in [(0, 0.0), (1, 0.0), (0, 1.0), (1, 1.0)]:
    run(128, 128, sym, beta, "3xtf32")
run(256, 128, 1, 1.0, "3xtf32")
