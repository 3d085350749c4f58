"""Isolated: fp32 sample-major patches + tf32 SYRK vs fp16 feature-major patches + f16 SYRK."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_15143_b200 import ops
dev = torch.device("cuda", 0)
SHAPES = [((32, 64, 56, 56), 3, 1, 1), ((32, 128, 28, 28), 3, 1, 1), ((32, 256, 14, 14), 3, 1, 1),
          ((32, 512, 7, 7), 3, 1, 1), ((32, 3, 224, 224), 7, 2, 3)]
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
for shape, k, s, p in SHAPES:
    x = torch.randn(shape, device=dev).contiguous(memory_format=torch.channels_last)
    op = ops.operand_im2col(x, (k, k), (s, s), (p, p), (1, 1), tap_major=k > 1)
    d, M = op.rows, op.cols
    out = torch.empty(d, d, device=dev)
    ld = (d + 3) // 4 * 4
    p32 = torch.empty(M, ld, device=dev)
    p16 = torch.empty(d, (M + 7) // 8 * 8, dtype=torch.float16, device=dev)
    m32 = t(lambda: ops.im2col_materialize([(op, p32)]))
    s32 = t(lambda: ops.syrk_ema([ops.factor_job(ops.operand_rows_mn(p32[:, :d]), out, 1.0 / M, 0.0)], "tf32"))
    m16 = t(lambda: ops.im2col_materialize_f16([(op, p16)]))
    s16 = t(lambda: ops.syrk_ema([ops.factor_job(ops.operand_rows_k_f16(p16, M), out, 1.0 / M, 0.0)], "tf32"))
    fl = d * (d + 1) * M
    print(f"{shape} k{k}: d={d} M={M} | f32: im2col {m32:.0f} us + syrk {s32:.0f} us ({fl/s32/1e6:.0f} TF/s) | "
          f"f16: im2col {m16:.0f} us + syrk {s16:.0f} us ({fl/s16/1e6:.0f} TF/s)", flush=True)
