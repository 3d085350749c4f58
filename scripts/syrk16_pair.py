"""One ResNet-50 3x3 layer's A-factor SYRK, fp16 implicit (TMA im2col) then fp16 patches,
3 launches each (ncu target).  python scripts/syrk16_pair.py C H"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import ops
c, h = int(sys.argv[1]), int(sys.argv[2])
x = torch.relu(torch.randn(32, c, h, h, device="cuda")).contiguous(memory_format=torch.channels_last)
op = ops.operand_im2col(x, (3, 3), (1, 1), (1, 1), (1, 1), tap_major=True)
out = torch.empty(op.rows, op.rows, device="cuda")
amax = torch.zeros(1, dtype=torch.int32, device="cuda")
x16 = torch.empty(32, h, h, c, dtype=torch.float16, device="cuda")
ops.im2col_materialize_f16([(op, x16, amax)])
ld = (op.cols + 7) // 8 * 8
p16 = torch.empty(op.rows, ld, dtype=torch.float16, device="cuda")
ops.im2col_materialize_f16([(op, p16, amax)])
for _ in range(3):
    ops.syrk_ema([ops.factor_job(ops.operand_im2col_f16(op, x16), out, 1.0 / op.cols, 0.0, x_amax=amax)], "tf32")
for _ in range(3):
    ops.syrk_ema([ops.factor_job(ops.operand_rows_k_f16(p16, op.cols), out, 1.0 / op.cols, 0.0, x_amax=amax)], "tf32")
torch.cuda.synchronize()
