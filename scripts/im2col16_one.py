"""fp16 patch materialization of one ResNet-50-like 3x3 conv (N=32, C, HxH, stride 1),
repeated: python scripts/im2col16_one.py C H [reps]  -- for ncu / timing."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import ops
c, h = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
x = torch.relu(torch.randn(32, c, h, h, device="cuda")).contiguous(memory_format=torch.channels_last)
op = ops.operand_im2col(x, (3, 3), (1, 1), (1, 1), (1, 1), tap_major=True)
d = op.rows
ld = (op.cols + 7) // 8 * 8
p16 = torch.empty(d, ld, dtype=torch.float16, device="cuda")
amax = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(2):
    ops.im2col_materialize_f16([(op, p16, amax)])
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps):
    ops.im2col_materialize_f16([(op, p16, amax)])
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
byts = d * op.cols * 2 + x.numel() * 4
print(f"C={c} H={h}: {ms*1e3:.1f} us per call (amax + patches), {byts/ms/1e6:.0f} GB/s (patch write + input read once)")
