"""Factored preconditioning (dpk_precond_factored) of the ResNet-50 layer set alone:
precond_one.py [reps] -> ms per call and useful TF/s (2(d_o^2 d_i + d_o d_i^2) per layer)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import ops
dev = torch.device("cuda", 0)
man = json.load(open(os.path.join(ROOT, "tests/golden/resnet50_manifest.json")))
torch.manual_seed(0)
jobs, keep, fl = [], [], 0.0
for d_in, d_out in man["dims"]:
    xa = torch.tril(torch.randn(d_in, ops.factor_ld(d_in), device=dev)[:, :d_in]) / d_in ** 0.5
    xg = torch.tril(torch.randn(d_out, ops.factor_ld(d_out), device=dev)[:, :d_out]) / d_out ** 0.5
    g = torch.randn(d_out, d_in, device=dev)
    out, tmp = torch.empty_like(g), torch.empty_like(g)
    keep += [xa, xg, g, out, tmp]
    jobs.append(ops.precond_factor_job(g, xa, xg, out, tmp))
    fl += 2.0 * (d_out * d_out * d_in + d_out * d_in * d_in)
ops.precondition_factored(jobs)
torch.cuda.synchronize()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    ops.precondition_factored(jobs)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
print(f"factored preconditioning of {len(jobs)} layers: {ms:.3f} ms, {fl / ms / 1e9:.1f} TF/s useful (3xTF32)")
