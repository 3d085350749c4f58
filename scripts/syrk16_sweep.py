"""f16 SYRK throughput on random fp16 K-major operands: d x M shapes, CUDA events,
median of reps; prints useful TF/s (lower triangle d(d+1)M flops).  Knobs come from
the environment (DPK_UNITS_PER_SM, DPK_SPLIT_MIN, DPK_CG2)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import ops
reps = 20
res = []
for d, M in ((576, 100352), (1152, 25088), (2304, 6272), (4608, 1568), (1024, 100352), (256, 401408)):
    p = torch.randn(d, M, device="cuda").half()
    out = torch.empty(d, d, device="cuda")
    job = ops.factor_job(ops.operand_rows_k_f16(p, M), out, 1.0 / M, 0.0)
    for _ in range(3):
        ops.syrk_ema([job], "tf32")
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); ops.syrk_ema([job], "tf32"); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    ms = ts[len(ts) // 2]
    res.append(f"{d}x{M}: {ms*1e3:.1f} us {d*(d+1)*M/ms/1e9:.0f} TF/s")
    del p
print(os.environ.get("TAG", ""), " | ".join(res), flush=True)
