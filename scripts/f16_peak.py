"""f16 tensor-core throughput of this engine (kind::f16, fp32 out) against cuBLAS
(torch.matmul half) on square N^3 and on a SYRK-like tall K: best of 10, CUDA events."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import _lib as L, ops


def best(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    b = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        b = min(b, s.elapsed_time(e))
    return b


for m, n, k in ((8192, 8192, 8192), (4096, 4096, 16384), (1024, 1024, 100352), (2048, 2048, 25088)):
    a = torch.randn(m, k, device="cuda").half()
    b = torch.randn(n, k, device="cuda").half()
    c = torch.empty(m, n, device="cuda")
    j = L.GemmJob()
    j.a, j.b = ops.operand_rows_k_f16(a, k), ops.operand_rows_k_f16(b, k)
    j.out, j.ldo, j.alpha = c.data_ptr(), n, 1.0
    t_dpk = best(lambda: ops.gemm([j], "tf32"))
    ch = torch.empty(m, n, device="cuda").half()
    t_cb = best(lambda: torch.matmul(a, b.t(), out=ch))
    f = 2.0 * m * n * k
    print(f"{m}x{n}x{k}: engine {f / t_dpk / 1e9:.0f} TF/s ({t_dpk*1e3:.0f} us), cuBLAS half {f / t_cb / 1e9:.0f} TF/s",
          flush=True)
