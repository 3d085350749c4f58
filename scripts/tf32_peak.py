"""Measured TF32 tensor-core peak on this B200 (the denominator of the bench's
tf32 roofline fractions; MEASURED_PEAKS.json only carries bf16).

  python scripts/tf32_peak.py [out.json]

Same method as the driver's bf16 number: 8192^3 fp32 matmul with TF32 math,
2*N^3 flops, best of 10 launches (burst) and back to back for ~4 s (sustained),
CUDA events.  Measured for cuBLAS (torch.matmul, allow_tf32) and for this
repo's own tcgen05 engine (dpk_gemm, 1-pass RN TF32 and 3xTF32).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2206_15143_b200 import _lib as L, ops  # noqa: E402

N = 8192
dev = torch.device("cuda", 0)
torch.backends.cuda.matmul.allow_tf32 = True
a = torch.randn(N, N, device=dev)
b = torch.randn(N, N, device=dev)
c = torch.empty(N, N, device=dev)
flops = 2.0 * N ** 3


def best_and_sustained(fn, secs=4.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    n, t0 = 0, time.perf_counter()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    while time.perf_counter() - t0 < secs:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    return flops / (best / 1e3) / 1e12, flops / (s.elapsed_time(e) / n / 1e3) / 1e12


out = {"n": N, "how": "8192^3 fp32 inputs, TF32 tensor-core math, 2*N^3 flops, best of 10 (burst) and "
                      "back to back for 4 s (sustained), CUDA events",
       "gpu": torch.cuda.get_device_name(dev)}
out["cublas_tf32_tflops"], out["cublas_tf32_tflops_sustained"] = best_and_sustained(lambda: torch.matmul(a, b, out=c))
bt = b.t().contiguous()  # engine operands: both K-major
j = L.GemmJob()
j.a, j.b = ops.operand_rows_k(a), ops.operand_rows_k(bt)
j.out, j.ldo, j.alpha = c.data_ptr(), N, 1.0
out["dpk_tf32_tflops"], out["dpk_tf32_tflops_sustained"] = best_and_sustained(lambda: ops.gemm([j], "tf32"))
out["dpk_3xtf32_tflops"], _ = best_and_sustained(lambda: ops.gemm([j], "3xtf32"), secs=0.5)
out["tf32_peak_tflops"] = max(out["cublas_tf32_tflops"], out["dpk_tf32_tflops"])
out["tf32_peak_tflops_sustained"] = max(out["cublas_tf32_tflops_sustained"], out["dpk_tf32_tflops_sustained"])
print(json.dumps(out, indent=1))
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
