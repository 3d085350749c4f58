import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import ops
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
src = []
for _ in range(cnt):
    x = torch.randn(n, n + 8, device=dev) / n ** 0.5
    src.append(x @ x.T)
dst = [torch.empty(n, n, device=dev) for _ in range(cnt)]
info = torch.zeros(cnt, dtype=torch.int32, device=dev)
jobs = [ops.spd_job(s, d, None, info[i:i + 1], 2) for i, (s, d) in enumerate(zip(src, dst))]
for _ in range(5):
    ops.chol_inv(jobs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    ops.chol_inv(jobs)
e1.record(); torch.cuda.synchronize()
print(f"leaf n={n} x{cnt}: {e0.elapsed_time(e1) / 20 * 1000:.1f} us per call; info {int(info.max())}; "
      f"err {float((src[0].double() @ dst[0].double() - torch.eye(n, device=dev, dtype=torch.float64)).norm()):.2e}")
