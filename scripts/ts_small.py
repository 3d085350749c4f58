"""Checkpoint timeline (ns, CTA 0) of small GEMM launches (run with DPK_DEBUG_TS=1)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2206_15143_b200 import _lib as L, ops

names = ["start", "setup", "tma_done", "gather_done", "mma_done", "epi_u0", "epi_last", "final_bar", "dealloc",
         "epi_tfull", "epi_ld0", "epi_st0", "mma_first_tma"]
lib = L.load()
for n, prec in [(128, "tf32"), (128, "3xtf32"), (1024, "tf32")]:
    a = torch.randn(n, n, device="cuda")
    o = torch.empty(n, n, device="cuda")
    j = L.GemmJob()
    j.a = ops.operand_rows_k(a)
    j.b = ops.operand_rows_k(a)
    j.out, j.ldo = o.data_ptr(), n
    j.alpha = 1.0
    for _ in range(3):
        ops.gemm([j], prec)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 16)()
    lib.dpk_debug_timestamps(buf)
    t0 = buf[0]
    print(n, prec, {names[i]: (buf[i] - t0) / 1000.0 for i in range(13) if buf[i] >= t0})

import time
a = torch.randn(128, 128, device="cuda"); o = torch.empty(128, 128, device="cuda")
j = L.GemmJob(); j.a = ops.operand_rows_k(a); j.b = ops.operand_rows_k(a); j.out, j.ldo = o.data_ptr(), 128; j.alpha = 1.0
for _ in range(10): ops.gemm([j], "tf32")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200): ops.gemm([j], "tf32")
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host per ops.gemm call: {(t1 - t)/200*1e6:.1f} us, incl drain {(t2 - t)/200*1e6:.1f} us")
arr = L.array(L.GemmJob, [j]); lb = L.load()
need = lb.dpk_gemm_workspace_bytes(arr, 1)
ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
t = time.perf_counter()
for _ in range(200): lb.dpk_gemm(arr, 1, ws.data_ptr(), need, 1, st)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host per raw dpk_gemm call: {(t1 - t)/200*1e6:.1f} us, incl drain {(t2 - t)/200*1e6:.1f} us")
