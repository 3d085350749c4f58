"""Host-side cost of DPKFAC.step() in the steady state (cProfile, top functions)."""
import os, sys, cProfile, pstats, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.nn.functional as F
import bench_models as BM
from paper_2206_15143_b200 import DPKFAC
dev = torch.device("cuda", 0)
ctor, batch, shape, classes = BM.WORKLOADS["resnet50"]
torch.manual_seed(0)
model = ctor().to(dev).to(memory_format=torch.channels_last)
kf = DPKFAC(model, gamma=0.002, inv_type="inverse", check_numerics="deferred")
x = torch.randn(batch, *shape, device=dev).contiguous(memory_format=torch.channels_last)
y = torch.randint(0, classes, (batch,), device=dev)
for _ in range(2):
    F.cross_entropy(model(x), y).backward(); kf.step()
F.cross_entropy(model(x), y).backward()
caps = {ly.index: (ly.a_in, ly.g_out, ly.batch) for ly in kf.owned}
def restore():
    for ly in kf.owned:
        ly.a_in, ly.g_out, ly.batch = caps[ly.index]
for _ in range(3):
    restore(); kf.step()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    restore(); kf.step()
host = (time.perf_counter() - t) / 10
torch.cuda.synchronize()
print(f"host per step {host*1e3:.2f} ms (deferred check: paced by the GPU)")
kf.check_numerics = False
for n in (1, 3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        restore(); kf.step()
    h = (time.perf_counter() - t) / n
    torch.cuda.synchronize()
    print(f"host enqueue per step (no numerics read, {n} steps) {h*1e3:.2f} ms")
kf.check_numerics = "deferred"
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    restore(); kf.step()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
