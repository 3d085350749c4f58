import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import _lib as L, ops, kfac as FK
def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1000
for n in [64, 128, 256, 512]:
    a = torch.randn(n, n, device="cuda"); o = torch.empty(n, n, device="cuda")
    j = L.GemmJob(); j.a = ops.operand_rows_k(a); j.b = ops.operand_rows_k(a); j.out, j.ldo = o.data_ptr(), n; j.alpha = 1.0
    for prec in ["tf32", "3xtf32"]:
        print(f"gemm n={n} {prec}: {timeit(lambda: ops.gemm([j], prec)):.1f} us")
for n in [16, 64, 128]:
    m = torch.randn(n, n + 3, device="cuda"); spd = m @ m.T / n + torch.eye(n, device="cuda")
    print(f"spd inv n={n}: {timeit(lambda: FK.sym_inverse(spd)):.1f} us (incl. host sync)")
torch.cuda.synchronize()
x = torch.zeros(1, device="cuda")
print(f"empty torch op: {timeit(lambda: x.add_(1)):.1f} us")
