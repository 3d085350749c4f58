"""e2e breakdown: train step without DP-KFAC, with it (early off/on)."""
import sys, os, time, faulthandler
faulthandler.dump_traceback_later(int(os.environ.get("TMO", "240")), exit=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.nn.functional as F
import bench_models as BM
from paper_2206_15143_b200 import DPKFAC

dev = torch.device("cuda", 0)
torch.backends.cudnn.benchmark = True
ctor, batch, shape, classes = BM.WORKLOADS[os.environ.get("MODEL", "resnet50")]
torch.manual_seed(0)
model = ctor().to(dev).to(memory_format=torch.channels_last)
opt = torch.optim.SGD(model.parameters(), lr=1e-3, momentum=0.9)
g = torch.Generator().manual_seed(1234)
xh = torch.randn(batch, *shape, generator=g).contiguous(memory_format=torch.channels_last).pin_memory()
yh = torch.randint(0, classes, (batch,), generator=g).pin_memory()

def run(kf, n=20, sync_each=True):
    def step():
        xb = xh.to(dev, non_blocking=True); yb = yh.to(dev, non_blocking=True)
        opt.zero_grad(set_to_none=False)
        loss = F.cross_entropy(model(xb), yb)
        loss.backward()
        if kf is not None:
            kf.step()
        opt.step()
        return loss.item() if sync_each else loss
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); s.record()
    for _ in range(n):
        step()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n, (time.perf_counter() - t0) * 1000 / n

print("no kfac      : %.2f ms (wall %.2f)" % run(None), flush=True)
for early in (False, True, "low"):
    kf = DPKFAC(model, gamma=0.002, xi=0.95, inv_type="inverse", check_numerics="deferred", early=bool(early))
    if early == "low":
        kf.early_priority = "low"
    print(f"kfac early={early}: %.2f ms (wall %.2f)" % run(kf), flush=True)
    print(f"  no per-step sync : %.2f ms" % run(kf, sync_each=False)[0], flush=True)
    kf.remove_hooks()
# host time of step() alone
kf = DPKFAC(model, gamma=0.002, xi=0.95, inv_type="inverse", check_numerics="deferred")
run(kf, 3)
F.cross_entropy(model(xh.to(dev)), yh.to(dev)).backward()
torch.cuda.synchronize()
t0 = time.perf_counter(); kf.step(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("host step() %.2f ms, until idle %.2f ms" % ((t1 - t0) * 1000, (t2 - t0) * 1000))
