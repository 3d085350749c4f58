"""Graph-mode factored SPD inverse (dpk_chol_factor_inv_batched) of the ResNet-50 factor set
(SPD_ONLY=n restricts to one size, SPD_COUNT=c to the first c): inv_factor_one.py [reps]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import json, torch
from paper_2206_15143_b200 import ops
dev = torch.device("cuda", 0)
man = json.load(open(os.path.join(ROOT, "tests/golden/resnet50_manifest.json")))
dims = [d for a, g in man["dims"] for d in (a, g)]
if os.environ.get("SPD_ONLY"):
    dims = [d for d in dims if d == int(os.environ["SPD_ONLY"])]
if os.environ.get("SPD_COUNT"):
    dims = dims[:int(os.environ["SPD_COUNT"])]
torch.manual_seed(0)
jobs, keep = [], []
for d in dims:
    x = torch.randn(d, 2 * d + 64, device=dev)
    s = x @ x.T / x.shape[1]
    o = torch.zeros(d, ops.factor_ld(d), device=dev)[:, :d]
    i = torch.zeros(1, dtype=torch.int32, device=dev); sh = torch.full((1,), 0.01, device=dev)
    keep += [s, o, i, sh]; jobs.append(ops.spd_factor_job(s, o, sh, i, 2))
ops.chol_factor_inv(jobs); torch.cuda.synchronize()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
for _ in range(reps): ops.chol_factor_inv(jobs)
en.record(); torch.cuda.synchronize()
print(f"factored inverse of {len(dims)} factors: {st.elapsed_time(en) / reps:.3f} ms")
