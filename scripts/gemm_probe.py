"""Engine throughput probe: rows_k x rows_k GEMM at several (M, N, K) vs cuBLAS tf32."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2206_15143_b200 import _lib as L, ops


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


torch.backends.cuda.matmul.allow_tf32 = True
for (m, n, k) in [(384, 640, 96), (300, 1000, 200), (4096, 4096, 256), (4096, 4096, 1024), (4096, 4096, 8192), (8192, 8192, 8192), (2048, 2048, 65536),
                  (1024, 1024, 262144)]:
    a = torch.randn(m, k, device="cuda")
    b = torch.randn(n, k, device="cuda")
    o = torch.empty(m, n, device="cuda")
    j = L.GemmJob()
    j.a = ops.operand_rows_k(a)
    j.b = ops.operand_rows_k(b)
    j.out, j.ldo = o.data_ptr(), n
    j.alpha = 1.0
    fl = 2.0 * m * n * k
    res = []
    ref = (a[:512].double() @ b[:512].double().T).float()
    for prec in ["tf32", "3xtf32"]:
        ms = timeit(lambda: ops.gemm([j], prec))
        err = float((o[:512, :512] - ref).norm() / ref.norm())
        res.append(f"{prec} {fl / ms / 1e9:6.1f} (err {err:.1e})")
    ms = timeit(lambda: torch.matmul(a, b.T, out=o))
    res.append(f"cublas-tf32 {fl / ms / 1e9:6.1f}")
    print(f"M={m} N={n} K={k}: " + "  ".join(res) + " TF/s", flush=True)
