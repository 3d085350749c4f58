"""Per-unit timeline of CTA 0 of one engine launch (DPK_DEBUG_TS=1): MMA start, first data,
last MMA issued, epilogue start/end, in us from the first unit's MMA start.
python scripts/unit_trace.py f16|tf32 [N]"""
import ctypes as C
import os, sys
os.environ["DPK_DEBUG_TS"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import _lib as L, ops
dt = sys.argv[1] if len(sys.argv) > 1 else "f16"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
if dt == "syrk16":  # python scripts/unit_trace.py syrk16 D M
    D, M = N, int(sys.argv[3])
    x = torch.randn(D, M, device="cuda").half()
    out = torch.empty(D, D, device="cuda")
    job = ops.factor_job(ops.operand_rows_k_f16(x, M), out, 1.0 / M, 0.0)
    run = lambda: ops.syrk_ema([job], "tf32")
else:
    a = torch.randn(N, N, device="cuda")
    b = torch.randn(N, N, device="cuda")
    c = torch.empty(N, N, device="cuda")
    j = L.GemmJob()
    if dt == "f16":
        a, b = a.half(), b.half()
        j.a, j.b = ops.operand_rows_k_f16(a, N), ops.operand_rows_k_f16(b, N)
    else:
        j.a, j.b = ops.operand_rows_k(a), ops.operand_rows_k(b)
    j.out, j.ldo, j.alpha = c.data_ptr(), N, 1.0
    run = lambda: ops.gemm([j], dt if dt in ("3xtf32", "3xf16") else "tf32")
for _ in range(3):
    run()
torch.cuda.synchronize()
buf = (C.c_ulonglong * 320)()
L.check(ops.lib().dpk_debug_unit_timestamps(buf), "ts")
t = [[buf[5 * i + k] for k in range(5)] for i in range(64)]
pw = t[63]
if pw[3]:
    print(f"producer (CTA 0, thread 0): {pw[3]} chunks, per chunk cycles: wait free stage {pw[0] / pw[3]:.0f}, "
          f"wait TMA {pw[1] / pw[3]:.0f}, convert {pw[2] / pw[3]:.0f}")
t = t[:63]
t0 = t[0][0]
print(dt, N)
for i, r in enumerate(t):
    if r[0] == 0 or r[0] < t0:
        break
    f = [(x - t0) / 1e3 for x in r]
    print(f"unit {i:2d}: mma {f[0]:8.2f} data {f[1]:8.2f} issued {f[2]:8.2f} | epi {f[3]:8.2f} -> {f[4]:8.2f}  "
          f"(mma span {f[2]-f[0]:6.2f}, epi {f[4]-f[3]:6.2f})")
