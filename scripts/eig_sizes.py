"""Per-size: native block Jacobi (dpk_syevd_batched) vs cuSOLVER (torch.linalg.eigh),
k matrices of size n at once; DPK_EIG_SWEEPS as set."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2206_15143_b200 import ops
dev = torch.device("cuda", 0)
for n, k in ((129, 4), (256, 8), (512, 8), (1024, 4), (2304, 2), (4608, 3)):
    torch.manual_seed(n)
    jobs = []
    for _ in range(k):
        x = torch.relu(torch.randn(n, max(64, n // 3), device=dev))
        s = x @ x.T / x.shape[1]
        jobs.append((s, torch.empty_like(s), torch.empty(n, device=dev), torch.zeros(1, dtype=torch.int32, device=dev)))
    ops.syevd(jobs, 'native'); torch.cuda.synchronize()
    t0 = time.perf_counter(); ops.syevd(jobs, 'native'); torch.cuda.synchronize(); tn = time.perf_counter() - t0
    jc = [(s, torch.empty_like(s), torch.empty(n, device=dev), None) for s, *_ in jobs]
    ops.syevd(jc, "cusolver"); torch.cuda.synchronize()
    t0 = time.perf_counter(); ops.syevd(jc, "cusolver"); torch.cuda.synchronize(); tc = time.perf_counter() - t0
    s, q, w, _ = jobs[0]
    a = s.double().cpu().numpy(); qq = q.double().cpu().numpy(); ww = w.double().cpu().numpy()
    ref = np.linalg.eigvalsh(a)[::-1]
    print(f"n={n} x{k}: native {tn*1e3:.1f} ms, cusolver (8 streams) {tc*1e3:.1f} ms; native: orth "
          f"{np.abs(qq.T@qq-np.eye(n)).max():.1e}, eig err {np.abs(ww-ref).max()/np.abs(ref).max():.1e}, "
          f"recon {np.linalg.norm(qq@np.diag(ww)@qq.T-a)/np.linalg.norm(a):.1e}", flush=True)
