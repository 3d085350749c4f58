"""Timeline of one overlapped DPKFAC.step (ResNet-50): CUDA events on both streams."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, torch.nn.functional as F
import bench_models as BM
from paper_2206_15143_b200 import DPKFAC
from paper_2206_15143_b200 import dpkfac as D
dev = torch.device("cuda", 0)
ctor, batch, shape, classes = BM.WORKLOADS["resnet50"]
torch.manual_seed(0)
model = ctor().to(dev).to(memory_format=torch.channels_last)
kf = DPKFAC(model, gamma=0.002, inv_type="inverse", check_numerics="deferred")
x = torch.randn(batch, *shape, device=dev).contiguous(memory_format=torch.channels_last)
y = torch.randint(0, classes, (batch,), device=dev)
ev = []
def mark(name):
    e = torch.cuda.Event(enable_timing=True); e.record(); ev.append((name, e))
orig_f, orig_i, orig_p = kf._factor_stage, kf._inverse_stage, kf._precondition_stage
def wrap(fn, tag):
    def g(layers, *a):
        who = f"class{next((i for i, c in enumerate(classes) if layers and layers[0] in c), -1)}"
        mark(f"{who}:{tag}:begin"); r = fn(layers, *a); mark(f"{who}:{tag}:end"); return r
    return g
kf._factor_stage = wrap(orig_f, "factors"); kf._inverse_stage = wrap(orig_i, "inverse"); kf._precondition_stage = wrap(orig_p, "precond")
for it in range(4):
    F.cross_entropy(model(x), y).backward()
    classes = kf._size_classes(kf.owned) if hasattr(kf, "owned") else [[]]
    torch.cuda.synchronize()
    ev.clear()
    mark("start")
    kf.step()
    mark("end")
    torch.cuda.synchronize()
t0 = ev[0][1]
for name, e in ev:
    print(f"{t0.elapsed_time(e):8.3f} ms  {name}")
print("classes:", [[ly.index for ly in c] for c in classes])
