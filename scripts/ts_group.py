"""Grouped tiny GEMMs (inversion-round shaped) timed inside a CUDA graph, plus the
CTA-0 checkpoint timeline (DPK_DEBUG_TS=1)."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import _lib as L, ops
names = ["start", "setup", "tma_done", "gather_done", "mma_done", "epi_u0", "epi_last", "final_bar", "dealloc",
         "epi_tfull", "epi_ld0", "epi_st0", "c0_stores_done", "c0_sts", "c0_lds", "c0_pre_store"]
lib = L.load()
dev = torch.device("cuda", 0)
for nprob, n, prec in [(1, 128, "tf32"), (1, 128, "3xtf32"), (32, 128, "3xtf32"), (84, 128, "3xtf32"), (84, 256, "3xtf32")]:
    keep, jobs = [], []
    for _ in range(nprob):
        a = torch.randn(n, n, device=dev); b = torch.randn(n, n, device=dev); o = torch.empty(n, n, device=dev)
        keep += [a, b, o]
        j = L.GemmJob(); j.a = ops.operand_rows_k(a); j.b = ops.operand_rows_k(b); j.out, j.ldo = o.data_ptr(), n; j.alpha = 1.0
        jobs.append(j)
    ops.gemm(jobs, prec); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(20): ops.gemm(jobs, prec)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    buf = (C.c_ulonglong * 16)(); lib.dpk_debug_timestamps(buf); t0 = buf[0]
    tl = {names[i]: round((buf[i] - t0) / 1000.0, 2) for i in range(16) if buf[i] >= t0}
    print(f"{nprob:3d} x {n}^3 {prec}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/launch (graph)  CTA0 {tl}", flush=True)
