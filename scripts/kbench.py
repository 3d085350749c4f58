"""Micro-benchmarks of the tcgen05 engine on isolated problem shapes (CUDA events)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

from paper_2206_15143_b200 import _lib as L
from paper_2206_15143_b200 import ops


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def syrk_case(name, op_fn, d, m, precision="tf32"):
    out = torch.empty(d, d, device="cuda")
    op = op_fn()
    ms = timeit(lambda: ops.syrk_ema([ops.factor_job(op, out, 1.0 / m, 0.0)], precision))
    tiles = ((d + 127) // 128) * ((d + 127) // 128 + 1) // 2
    mma_flops = tiles * 128 * 128 * 2.0 * ((m + 31) // 32 * 32)
    uniq = d * (d + 1) * float(m)
    print(f"{name:38s} d={d:5d} M={m:7d} {precision:6s} {ms:8.3f} ms  unique {uniq / ms / 1e9:7.1f} TF/s  "
          f"tile-MMA {mma_flops / ms / 1e9:7.1f} TF/s", flush=True)


def main():
    torch.manual_seed(0)
    dev = torch.device("cuda", 0)
    # plain K-major rows (like NCHW 1x1 slabs / inversion operands)
    for d, m in [(1024, 65536), (512, 100352), (4608, 1568), (128, 401408)]:
        x = torch.randn(d, m, device=dev)
        syrk_case("rows_k", lambda: ops.operand_rows_k(x), d, m)
        syrk_case("rows_k", lambda: ops.operand_rows_k(x), d, m, "3xtf32")
    # sample-major (nn.Linear input)
    for d, m in [(1024, 65536), (4608, 1568), (576, 100352), (2304, 6272), (1152, 25088)]:
        x = torch.randn(m, d, device=dev)
        syrk_case("rows_mn", lambda: ops.operand_rows_mn(x), d, m)
        x = torch.randn(d, m, device=dev)
        syrk_case("rows_k", lambda: ops.operand_rows_k(x), d, m)
    # implicit im2col, ResNet-50 shapes
    for (c, h, k, s, p) in [(64, 56, 3, 1, 1), (128, 28, 3, 1, 1), (256, 14, 3, 1, 1), (512, 7, 3, 1, 1),
                            (64, 56, 1, 1, 0), (3, 224, 7, 2, 3), (256, 56, 1, 2, 0)]:
        xin = torch.relu(torch.randn(32, c, h, h, device=dev))
        op = ops.operand_im2col(xin, (k, k), (s, s), (p, p), (1, 1))
        syrk_case(f"im2col c{c} {h}x{h} k{k} s{s}", lambda: op, op.rows, op.cols)
    # general GEMM 3xTF32 (inversion-style)
    for n in [4608, 2304, 1152]:
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        o = torch.empty(n, n, device=dev)
        j = L.GemmJob()
        j.a, j.b = ops.operand_rows_k(a), ops.operand_rows_k(b)
        j.out, j.ldo = o.data_ptr(), n
        j.alpha = 1.0
        for prec in ("tf32", "tf32-trunc", "3xtf32"):
            ms = timeit(lambda: ops.gemm([j], prec))
            print(f"gemm rows_k x rows_k n={n} {prec:6s} {ms:8.3f} ms  {2.0 * n ** 3 / ms / 1e9:7.1f} TF/s", flush=True)
        j.b = ops.operand_rows_mn(b)
        ms = timeit(lambda: ops.gemm([j], "3xtf32"))
        print(f"gemm rows_k x rows_mn n={n} 3xtf32 {ms:8.3f} ms  {2.0 * n ** 3 / ms / 1e9:7.1f} TF/s", flush=True)
    # cuBLAS reference points
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(8192, 8192, device=dev)
    ms = timeit(lambda: a @ a)
    print(f"cuBLAS tf32 8192^3 {ms:8.3f} ms {2.0 * 8192 ** 3 / ms / 1e9:7.1f} TF/s")


if __name__ == "__main__":
    main()
