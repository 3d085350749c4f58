"""Per-layer factor SYRK timing on ResNet-50 captures (channels_last unless --nchw)."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, torch.nn.functional as F
import bench_models as BM
from paper_2206_15143_b200 import DPKFAC, ops

ap = argparse.ArgumentParser(); ap.add_argument("--nchw", action="store_true"); ap.add_argument("--model", default="resnet50")
ap.add_argument("--im2col", default="materialize")
args = ap.parse_args()
dev = torch.device("cuda", 0)
ctor, batch, shape, classes = BM.WORKLOADS[args.model]
torch.manual_seed(0)
mf = torch.contiguous_format if args.nchw else torch.channels_last
model = ctor().to(dev).to(memory_format=mf)
kf = DPKFAC(model, inv_type="inverse")
x = torch.randn(batch, *shape, device=dev).contiguous(memory_format=mf)
y = torch.randint(0, classes, (batch,), device=dev)
F.cross_entropy(model(x), y).backward()
rows = []
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
mat_ms = 0.0
for ly in kf.owned:
    oa, pending = ly.operand_a(args.im2col)
    if pending is not None:
        ms = t(lambda: ops.im2col_materialize([pending]))
        mat_ms += ms
        rows.append((ms, ly.index, ly.name, "P", pending[0].rows, pending[0].cols, -1, 0.0))
    for side, op, d in (("A", oa, ly.d_in), ("G", ly.operand_g(), ly.d_out)):
        out = torch.empty(d, d, device=dev)
        ms = t(lambda: ops.syrk_ema([ops.factor_job(op, out, 1.0 / op.cols, 0.0)], "tf32"))
        flops = d * (d + 1) * op.cols
        rows.append((ms, ly.index, ly.name, side, d, op.cols, op.kind, flops / ms / 1e9))
tot = sum(r[0] for r in rows)
print(f"sum of isolated ops {tot:.2f} ms (materialize {mat_ms:.2f} ms)")
for r in sorted(rows, reverse=True)[:16]:
    print(f"{r[0]:7.3f} ms  L{r[1]:2d} {r[2]:24s} {r[3]} d={r[4]:5d} M={r[5]:7d} kind={r[6]} {r[7]:7.1f} TF/s")
