"""TRI-mode leaf (the SPD recursion's diagonal blocks): n = 128 blocks of 4608 matrices,
cnt leaves in one launch.  leaf_tri.py [cnt]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import ops
cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
# n = 256 matrices -> recursion 128 + 128: the first round is cnt TRI leaves of 128
src, dst = [], []
for _ in range(cnt):
    x = torch.randn(256, 300, device=dev) / 17.0
    src.append(x @ x.T)
    dst.append(torch.empty(256, 256, device=dev))
info = torch.zeros(cnt, dtype=torch.int32, device=dev)
jobs = [ops.spd_job(s, d, None, info[i:i + 1], 2) for i, (s, d) in enumerate(zip(src, dst))]
for _ in range(3):
    ops.chol_inv(jobs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    ops.chol_inv(jobs)
e1.record(); torch.cuda.synchronize()
print(f"n=256 x{cnt} inverse: {e0.elapsed_time(e1) / 10 * 1000:.1f} us per call")
