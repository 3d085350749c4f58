"""Native block-Jacobi eigensolver (csrc/syevj.cu) on the ResNet-50 factor set (or
SPD_ONLY=n): time per batched call + accuracy against float64 eigh on a sample."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import json, numpy as np, torch
from paper_2206_15143_b200 import ops
dev = torch.device("cuda", 0)
man = json.load(open(os.path.join(ROOT, "tests/golden/resnet50_manifest.json")))
dims = [d for a, g in man["dims"] for d in (a, g)]
if os.environ.get("SPD_ONLY"):
    dims = [d for d in dims if d == int(os.environ["SPD_ONLY"])]
torch.manual_seed(0)
jobs = []
for d in dims:
    x = torch.relu(torch.randn(d, max(64, d // 3), device=dev))
    s = x @ x.T / x.shape[1]
    jobs.append((s, torch.empty_like(s), torch.empty(d, device=dev), torch.zeros(1, dtype=torch.int32, device=dev)))
ops.syevd(jobs); torch.cuda.synchronize()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
t0 = time.perf_counter()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
for _ in range(reps): ops.syevd(jobs)
en.record(); torch.cuda.synchronize()
print(f"eigendecomposition of {len(dims)} factors (n > 128: {sum(d > 128 for d in dims)}): "
      f"{st.elapsed_time(en) / reps:.2f} ms/call, sweeps={os.environ.get('DPK_EIG_SWEEPS', '8')}")
worst = {}
for s, q, w, info in jobs[::7]:
    n = s.shape[0]
    a = s.double().cpu().numpy(); qq = q.double().cpu().numpy(); ww = w.double().cpu().numpy()
    ref = np.linalg.eigvalsh(a)[::-1]
    e1 = np.abs(ww - ref).max() / np.abs(ref).max()
    e2 = np.abs(qq.T @ qq - np.eye(n)).max()
    e3 = np.linalg.norm(qq @ np.diag(ww) @ qq.T - a) / np.linalg.norm(a)
    worst[n] = (f"{e1:.1e}", f"{e2:.1e}", f"{e3:.1e}", int(info.item()))
print("n: (eigval err, orthogonality, reconstruction, info)", worst)
