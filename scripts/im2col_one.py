import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import ops
c, h = int(sys.argv[1]), int(sys.argv[2])
x = torch.relu(torch.randn(32, c, h, h, device="cuda")).contiguous(memory_format=torch.channels_last)
op = ops.operand_im2col(x, (3, 3), (1, 1), (1, 1), (1, 1), tap_major=True)
out = torch.empty(op.rows, op.rows, device="cuda")
for _ in range(3):
    ops.syrk_ema([ops.factor_job(op, out, 1.0 / op.cols, 0.0)], "tf32")
torch.cuda.synchronize()
