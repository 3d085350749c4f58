"""Isolated factor SYRK: tiled-TMA tap boxes (implicit, kind::tf32) vs materialized fp32
patches (MN3, kind::tf32) vs the default prescaled fp16 patches (kind::f16)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_15143_b200 import ops
dev = torch.device("cuda", 0)
SHAPES = [((32, 64, 56, 56), 3, 1, 1), ((32, 128, 56, 56), 3, 2, 1), ((32, 128, 28, 28), 3, 1, 1),
          ((32, 256, 14, 14), 3, 1, 1), ((32, 512, 7, 7), 3, 1, 1), ((32, 256, 56, 56), 1, 2, 0)]
only = os.environ.get("ONLY")
for i, (shape, k, s, p) in enumerate(SHAPES):
    if only is not None and int(only) != i:
        continue
    x = torch.randn(shape, device=dev).contiguous(memory_format=torch.channels_last)
    op = ops.operand_im2col(x, (k, k), (s, s), (p, p), (1, 1), tap_major=True)
    d, M = op.rows, op.cols
    out = torch.empty(d, d, device=dev)
    ld = (d + 3) // 4 * 4
    patch = torch.empty(M, ld, device=dev)
    p16 = torch.empty(d, (M + 7) // 8 * 8, dtype=torch.float16, device=dev)
    amax = torch.zeros(1, dtype=torch.int32, device=dev)
    res = {}
    for mode in ("taps", "mat", "f16"):
        def run():
            if mode == "taps":
                ops.syrk_ema([ops.factor_job(op, out, 1.0 / M, 0.0)], "tf32")
            elif mode == "f16":
                ops.im2col_materialize_f16([(op, p16, amax)])
                ops.syrk_ema([ops.factor_job(ops.operand_rows_k_f16(p16, M), out, 1.0 / M, 0.0, x_amax=amax)], "tf32")
            else:
                ops.im2col_materialize([(op, patch)])
                ops.syrk_ema([ops.factor_job(ops.operand_rows_mn(patch[:, :d]), out, 1.0 / M, 0.0)], "tf32")
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            run()
        b.record()
        torch.cuda.synchronize()
        res[mode] = a.elapsed_time(b) / 10
    fl = d * (d + 1) * M
    print(f"{shape} k{k} s{s}: d={d} M={M}  taps {res['taps']*1e3:.1f} us ({fl/res['taps']/1e9:.0f} TF/s)  "
          f"fp32 patches+syrk {res['mat']*1e3:.1f} us  fp16 patches+f16 syrk {res['f16']*1e3:.1f} us", flush=True)
