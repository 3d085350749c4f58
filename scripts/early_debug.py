import sys, os, time, faulthandler
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(int(os.environ.get("TMO", "90")), exit=True)
import torch, torch.nn.functional as F
import bench_models as BM
from paper_2206_15143_b200 import DPKFAC
dev = torch.device("cuda", 0)
ctor, batch, shape, classes = BM.WORKLOADS[os.environ.get("MODEL", "resnet50")]
torch.manual_seed(0)
model = ctor().to(dev).to(memory_format=torch.channels_last)
x = torch.randn(batch, *shape, device=dev).contiguous(memory_format=torch.channels_last)
y = torch.randint(0, classes, (batch,), device=dev)
kf = DPKFAC(model, gamma=0.002, xi=0.95, inv_type="inverse", check_numerics=os.environ.get("CHK", "deferred"), early=True)
for it in range(4):
    print("iter", it, "fwd", flush=True)
    loss = F.cross_entropy(model(x), y)
    print("iter", it, "bwd", flush=True)
    loss.backward()
    print("iter", it, "bwd done; launched", kf._launched, flush=True)
    torch.cuda.synchronize()
    print("iter", it, "synced", flush=True)
    kf.step()
    torch.cuda.synchronize()
    print("iter", it, "step done", flush=True)
print("ok")
