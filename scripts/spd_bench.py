"""SPD inverse (K3) on the ResNet-50 factor set: all 108 damped factors of one
step in one batched call; DPK_SPD_TRACE=1 prints the per-round table."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import json
import torch
from paper_2206_15143_b200 import ops

dev = torch.device("cuda", 0)
man = json.load(open(os.path.join(ROOT, "tests/golden/resnet50_manifest.json")))
dims = []
for a, g in man["dims"]:
    dims += [a, g]
only = os.environ.get("SPD_ONLY")
if only:
    dims = [d for d in dims if d == int(only)]
torch.manual_seed(0)
srcs, dsts, infos, shifts = [], [], [], []
for d in dims:
    x = torch.randn(d, 2 * d + 64, device=dev)
    srcs.append(x @ x.T / x.shape[1])
    dsts.append(torch.empty(d, d, device=dev))
    infos.append(torch.zeros(1, dtype=torch.int32, device=dev))
    shifts.append(torch.full((1,), 0.01, device=dev))
jobs = [ops.spd_job(s, o, sh, i, 2) for s, o, sh, i in zip(srcs, dsts, shifts, infos)]
ops.chol_inv(jobs)
torch.cuda.synchronize()
if os.environ.get("DPK_SPD_TRACE") == "1":
    sys.exit(0)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    ops.chol_inv(jobs)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
fl = sum(float(d) ** 3 for d in dims)
print(f"{len(dims)} factors, {ms:.3f} ms, {fl / ms / 1e9:.1f} TF/s (n^3 convention)")
for d in (4608, 2049, 576):
    idx = dims.index(d) if d in dims else None
    if idx is None: continue
    a = srcs[idx].double() + 0.01 * torch.eye(d, device=dev, dtype=torch.float64)
    err = (dsts[idx].double() @ a - torch.eye(d, device=dev, dtype=torch.float64)).norm() / d ** 0.5
    print(f"n={d}: ||X A - I||_F/sqrt(n) = {err:.2e}")
