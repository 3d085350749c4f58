"""On-chip Jacobi (n <= 128) cost and accuracy: k matrices of n, rank r (DPK_JAC_REL/ABS knobs)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2206_15143_b200 import ops
n, k, r = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda", 0)
torch.manual_seed(0)
jobs = []
for _ in range(k):
    x = torch.relu(torch.randn(n, r, device=dev))
    s = x @ x.T / r
    jobs.append((s, torch.empty_like(s), torch.empty(n, device=dev), torch.zeros(1, dtype=torch.int32, device=dev)))
ops.syevd(jobs, "native"); torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record(); ops.syevd(jobs, "native"); en.record(); torch.cuda.synchronize()
s, q, w, _ = jobs[0]
a = s.double().cpu().numpy(); qq = q.double().cpu().numpy(); ww = w.double().cpu().numpy()
ref = np.linalg.eigvalsh(a)[::-1]
print(f"n={n} k={k} rank={r} rel={os.environ.get("DPK_JAC_REL","2e-6")}: {st.elapsed_time(en)*1e3:.0f} us, "
      f"eig err {np.abs(ww-ref).max()/np.abs(ref).max():.1e}, orth {np.abs(qq.T@qq-np.eye(n)).max():.1e}, "
      f"recon {np.linalg.norm(qq@np.diag(ww)@qq.T-a)/np.linalg.norm(a):.1e}")
