"""Per-phase cycle split of the SPD leaf sweep (needs scripts/micro/libdpkfac_prof.so, built with -DDPK_LEAF_PROF)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DPK_SPD_GRAPH"] = "0"
from paper_2206_15143_b200 import _lib as L

PROF = os.path.join(ROOT, "scripts", "micro", "libdpkfac_prof.so")
L.load(PROF)
import torch

from paper_2206_15143_b200 import ops

dev = torch.device("cuda", 0)
cnt = 3
src = [(lambda x: x @ x.T)(torch.randn(256, 300, device=dev) / 17.0) for _ in range(cnt)]
dst = [torch.empty(256, 256, device=dev) for _ in range(cnt)]
info = torch.zeros(cnt, dtype=torch.int32, device=dev)
jobs = [ops.spd_job(s, d, None, info[i:i + 1], 2) for i, (s, d) in enumerate(zip(src, dst))]
ops.chol_inv(jobs)
torch.cuda.synchronize()
lib = C.CDLL(PROF)
buf = (C.c_ulonglong * 12)()
lib.dpk_leaf_prof(buf)
for t, off in (("thread 0", 0), ("thread 511", 6)):
    n = max(buf[off + 5], 1)
    print(t, "steps", buf[off + 5], "avg cycles: publish %d, bar1 %d, phase2 %d, bar2 %d, phase3 %d" %
          tuple(buf[off + i] // n for i in range(5)))
