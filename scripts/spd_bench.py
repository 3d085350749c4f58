"""Batched damped SPD inverse over the ResNet-50 factor sizes (54 layers -> 108
matrices), timed alone with CUDA events; DPK_SPD_TRACE=1 adds the per-round table."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2206_15143_b200 import ops

dims = json.load(open(os.path.join(ROOT, "tests/golden/resnet50_manifest.json")))["dims"]
only = int(sys.argv[1]) if len(sys.argv) > 1 else 0
ns = [n for p in dims for n in p if n > only]
dev = torch.device("cuda", 0)
torch.manual_seed(0)
src, dst = [], []
for n in ns:
    x = torch.randn(n, n + 64, device=dev) / (n + 64) ** 0.5
    src.append(x @ x.T)
    dst.append(torch.empty(n, n, device=dev))
shift = torch.full((1,), 1e-3, device=dev)
info = torch.zeros(len(ns), dtype=torch.int32, device=dev)
jobs = [ops.spd_job(s, d, shift, info[i:i + 1], 2) for i, (s, d) in enumerate(zip(src, dst))]
for _ in range(3):
    ops.chol_inv(jobs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    ops.chol_inv(jobs)
e1.record()
torch.cuda.synchronize()
print(f"{len(ns)} matrices (n > {only}): {e0.elapsed_time(e1) / reps:.3f} ms per batched inverse; info max {int(info.max())}")
i = max(range(len(ns)), key=lambda k: ns[k])
eye = torch.eye(ns[i], device=dev, dtype=torch.float64)
a = src[i].double() + 1e-3 * eye
print(f"largest n={ns[i]}: |A X - I|_F / sqrt(n) = {float(torch.linalg.norm(a @ dst[i].double() - eye) / ns[i] ** 0.5):.2e}")
if os.environ.get("TRACE_ONCE"):
    os.environ["DPK_SPD_TRACE"] = "1"
