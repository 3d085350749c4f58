"""e2e split: training iteration without DP-KFAC, with its capture hooks only (no
step()), and with step(): python scripts/e2e_hooks.py [model]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.nn.functional as F
import bench_models as BM
from paper_2206_15143_b200 import DPKFAC

dev = torch.device("cuda", 0)
torch.backends.cudnn.benchmark = True
name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
ctor, batch, shape, classes = BM.WORKLOADS[name]
torch.manual_seed(0)
model = ctor().to(dev).to(memory_format=torch.channels_last)
opt = torch.optim.SGD(model.parameters(), lr=1e-3, momentum=0.9)
xh = torch.randn(batch, *shape).contiguous(memory_format=torch.channels_last).pin_memory()
yh = torch.randint(0, classes, (batch,)).pin_memory()


def run(kf, do_step, n=20):
    def it():
        xb = xh.to(dev, non_blocking=True); yb = yh.to(dev, non_blocking=True)
        opt.zero_grad(set_to_none=False)
        loss = F.cross_entropy(model(xb), yb)
        loss.backward()
        if do_step:
            kf.step()
        opt.step()
        return loss.item()
    for _ in range(3):
        it()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); s.record()
    for _ in range(n):
        it()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n, (time.perf_counter() - t0) * 1000 / n


print(f"{name} no kfac         : %.2f ms (wall %.2f)" % run(None, False), flush=True)
kf = DPKFAC(model, gamma=0.002, xi=0.95, inv_type="inverse", check_numerics="deferred", assignment="balanced")
print(f"{name} hooks, no step(): %.2f ms (wall %.2f)" % run(kf, False), flush=True)
print(f"{name} hooks + step()  : %.2f ms (wall %.2f)" % run(kf, True), flush=True)
# host-side cost of the forward + backward alone (CPU time until the last launch)
for label in ("hooks", "no kfac"):
    if label == "no kfac":
        kf.remove_hooks()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    loss = F.cross_entropy(model(xh.to(dev, non_blocking=True)), yh.to(dev, non_blocking=True))
    t1 = time.perf_counter()
    loss.backward()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{name} host ({label}): forward issue %.2f ms, backward issue %.2f ms, until idle %.2f ms"
          % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t0) * 1e3), flush=True)
