"""Per-layer factor cost of the ResNet-50 3x3 convs (N=32): fp16 patch route
(amax + patches + kind::f16 SYRK) against the implicit-im2col SYRKs, CUDA events,
median of reps.  python scripts/implicit_vs_f16.py [reps]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import ops

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for c, h in ((64, 56), (128, 28), (256, 14), (512, 7)):
    x = torch.relu(torch.randn(32, c, h, h, device="cuda")).contiguous(memory_format=torch.channels_last)
    op = ops.operand_im2col(x, (3, 3), (1, 1), (1, 1), (1, 1), tap_major=True)
    d = op.rows
    out = torch.empty(d, d, device="cuda")
    ld = (op.cols + 7) // 8 * 8
    p16 = torch.empty(d, ld, dtype=torch.float16, device="cuda")
    amax = torch.zeros(1, dtype=torch.int32, device="cuda")
    op16 = ops.operand_rows_k_f16(p16, op.cols)

    def f16_route():
        ops.im2col_materialize_f16([(op, p16, amax)])
        ops.syrk_ema([ops.factor_job(op16, out, 1.0 / op.cols, 0.0, x_amax=amax)], "tf32")

    def f16_syrk():
        ops.syrk_ema([ops.factor_job(op16, out, 1.0 / op.cols, 0.0, x_amax=amax)], "tf32")

    x16 = torch.empty(32, h, h, c, dtype=torch.float16, device="cuda")
    op_i16 = ops.operand_im2col_f16(op, x16)

    def implicit16():
        ops.im2col_materialize_f16([(op, x16, amax)])
        ops.syrk_ema([ops.factor_job(op_i16, out, 1.0 / op.cols, 0.0, x_amax=amax)], "tf32")

    def implicit16_syrk():
        ops.syrk_ema([ops.factor_job(op_i16, out, 1.0 / op.cols, 0.0, x_amax=amax)], "tf32")

    def implicit():
        ops.syrk_ema([ops.factor_job(op, out, 1.0 / op.cols, 0.0)], "tf32")

    # DPK_TAPS=0 in the environment selects the TMA im2col-mode form for "implicit"
    r = {"f16 route": timed(f16_route), "f16 syrk only": timed(f16_syrk), "implicit fp32": timed(implicit),
         "implicit16 route": timed(implicit16), "implicit16 syrk only": timed(implicit16_syrk)}
    print(f"C={c} H={h} d={d} M={op.cols}: " + ", ".join(f"{k} {v:.1f} us" for k, v in r.items()), flush=True)
