"""One factor SYRK (F = alpha X X^T + beta F):  syrk_one.py d M [k|mn] [reps] [beta]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import ops
d, m = int(sys.argv[1]), int(sys.argv[2])
lay = sys.argv[3] if len(sys.argv) > 3 else "k"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
beta = float(sys.argv[5]) if len(sys.argv) > 5 else 0.05
dev = torch.device("cuda", 0)
if lay == "k":
    x = torch.randn(d, m, device=dev); op = ops.operand_rows_k(x)
else:
    x = torch.randn(m, d, device=dev); op = ops.operand_rows_mn(x)
out = torch.zeros(d, d, device=dev)
job = [ops.factor_job(op, out, 1.0 / m, beta)]
ops.syrk_ema(job, "tf32"); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps): ops.syrk_ema(job, "tf32")
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
print(f"SYRK d={d} M={m} {lay}: {ms*1e3:.1f} us  {d*(d+1)*m/ms/1e9:.1f} TF/s unique")
