"""Host-side cost of DPKFAC.step() for a bench model: wall time of the Python call
without syncs, and the cProfile top entries.  python scripts/host_time_model.py [model]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, torch.nn.functional as F
import bench_models as BM
from paper_2206_15143_b200 import DPKFAC
name = sys.argv[1] if len(sys.argv) > 1 else "densenet201"
dev = torch.device("cuda", 0)
ctor, batch, shape, classes = BM.WORKLOADS[name]
torch.manual_seed(0)
model = ctor().to(dev).to(memory_format=torch.channels_last)
kf = DPKFAC(model, gamma=0.002, inv_type="inverse", check_numerics="deferred", assignment="balanced")
x = torch.randn(batch, *shape, device=dev).contiguous(memory_format=torch.channels_last)
y = torch.randint(0, classes, (batch,), device=dev)
for i in range(5):
    F.cross_entropy(model(x), y).backward()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kf.step()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name} step {i}: host {1e3*(t1-t0):.2f} ms, host+drain {1e3*(t2-t0):.2f} ms")
import cProfile, pstats
F.cross_entropy(model(x), y).backward(); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable(); kf.step(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
