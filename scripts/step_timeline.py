"""Per-class timeline of one overlapped DPKFAC.step() (ResNet-50, B=32, inverse mode):
CUDA events around every stage call on the stream it runs on, printed in us from the
step's first event.  python scripts/step_timeline.py [model]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import torch.nn.functional as F

import bench_models as BM
from paper_2206_15143_b200 import DPKFAC

model_name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
dev = torch.device("cuda", 0)
ctor, batch, shape, classes = BM.WORKLOADS[model_name]
torch.manual_seed(0)
model = ctor().to(dev).to(memory_format=torch.channels_last)
kf = DPKFAC(model, gamma=0.002, xi=0.95, inv_type="inverse", assignment="balanced", check_numerics="deferred")
if os.environ.get("SIDE_CAP"):
    kf.SIDE_CAP = int(os.environ["SIDE_CAP"])
x = torch.randn(batch, *shape, device=dev).contiguous(memory_format=torch.channels_last)
y = torch.randint(0, classes, (batch,), device=dev)
F.cross_entropy(model(x), y).backward()
kf.step()
model.zero_grad(set_to_none=False)
F.cross_entropy(model(x), y).backward()
saved = {ly.index: (ly.a_in, ly.g_out, ly.batch) for ly in kf.owned}
params = [p for ly in kf.layers for p in ([ly.module.weight] + ([ly.module.bias] if ly.has_bias else []))]
grads = [p.grad.clone() for p in params]


def restore():
    for ly in kf.owned:
        ly.a_in, ly.g_out, ly.batch = saved[ly.index]
    torch._foreach_copy_([p.grad for p in params], grads)


marks = []


def wrap(name):
    orig = getattr(kf, name)

    def f(layers, *a, **k):
        st = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        r = orig(layers, *a, **k)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(st)
        marks.append((name[1:], len(layers), max(max(l.d_in, l.d_out) for l in layers) if layers else 0,
                      st.stream_id, e0, e1))
        return r
    setattr(kf, name, f)


for n in ("_factor_stage", "_inverse_stage", "_precondition_stage"):
    wrap(n)
for _ in range(5):
    restore()
    kf.step()
torch.cuda.synchronize()
marks.clear()
restore()
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
kf.step()
t1 = torch.cuda.Event(enable_timing=True)
t1.record()
torch.cuda.synchronize()
print(f"{model_name}: step {t0.elapsed_time(t1) * 1e3:.0f} us")
for name, n, dmax, sid, e0, e1 in marks:
    print(f"  {name:18s} layers={n:3d} max_d={dmax:5d} stream={sid:3d}  {t0.elapsed_time(e0) * 1e3:8.0f} -> "
          f"{t0.elapsed_time(e1) * 1e3:8.0f}  ({e0.elapsed_time(e1) * 1e3:7.0f} us)")
kf.check()
