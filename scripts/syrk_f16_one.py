"""One factor SYRK of layer1.x.conv2's A (576 x 100352) on fp16 patches (kind::f16) or
fp32 patches (kind::tf32): syrk_f16_one.py f16|f32 (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_15143_b200 import ops
dev = torch.device("cuda", 0)
mode = sys.argv[1] if len(sys.argv) > 1 else "f16"
x = torch.randn(32, 64, 56, 56, device=dev).contiguous(memory_format=torch.channels_last)
op = ops.operand_im2col(x, (3, 3), (1, 1), (1, 1), (1, 1), tap_major=True)
d, M = op.rows, op.cols
out = torch.empty(d, d, device=dev)
if mode == "f16":
    p = torch.empty(d, (M + 7) // 8 * 8, dtype=torch.float16, device=dev)
    ops.im2col_materialize_f16([(op, p)])
    job = ops.factor_job(ops.operand_rows_k_f16(p, M), out, 1.0 / M, 0.0)
else:
    p = torch.empty(M, (d + 3) // 4 * 4, device=dev)
    ops.im2col_materialize([(op, p)])
    job = ops.factor_job(ops.operand_rows_mn(p[:, :d]), out, 1.0 / M, 0.0)
for _ in range(3):
    ops.syrk_ema([job], "tf32")
torch.cuda.synchronize()
print("ok")
