"""fp16 patches of the ResNet-50 stem (N=32, 3x224x224, 7x7/2 pad 3), repeated."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import ops
x = torch.randn(32, 3, 224, 224, device="cuda").contiguous(memory_format=torch.channels_last)
op = ops.operand_im2col(x, (7, 7), (2, 2), (3, 3), (1, 1), tap_major=True)
p16 = torch.empty(op.rows, (op.cols + 7) // 8 * 8, dtype=torch.float16, device="cuda")
amax = torch.zeros(1, dtype=torch.int32, device="cuda")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for _ in range(3): ops.im2col_materialize_f16([(op, p16, amax)])
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps): ops.im2col_materialize_f16([(op, p16, amax)])
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
print(f"stem fp16 patches {op.rows}x{op.cols}: {ms*1e3:.1f} us per call (amax + patches), {op.rows*op.cols*2/ms/1e6:.0f} GB/s written")
