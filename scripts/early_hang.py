import sys, os, time, faulthandler
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(int(os.environ.get("TMO", "60")), exit=True)
import torch, torch.nn.functional as F
import bench_models as BM
from paper_2206_15143_b200 import DPKFAC
dev = torch.device("cuda", 0)
torch.backends.cudnn.benchmark = True
ctor, batch, shape, classes = BM.WORKLOADS["resnet50"]
torch.manual_seed(0)
model = ctor().to(dev).to(memory_format=torch.channels_last)
opt = torch.optim.SGD(model.parameters(), lr=1e-3, momentum=0.9)
x = torch.randn(batch, *shape, device=dev).contiguous(memory_format=torch.channels_last)
y = torch.randint(0, classes, (batch,), device=dev)
kf = DPKFAC(model, gamma=0.002, xi=0.95, inv_type="inverse", check_numerics="deferred", early=os.environ.get("EARLY", "1") == "1")
only = os.environ.get("ONLY")
t0 = time.time()
for it in range(int(os.environ.get("ITERS", "30"))):
    opt.zero_grad(set_to_none=False)
    loss = F.cross_entropy(model(x), y)
    loss.backward()
    if only is not None:
        kf._launched = {k: v for k, v in kf._launched.items()}
    kf.step()
    opt.step()
    loss.item()
print("ok", os.environ.get("TAG"), "%.2f ms/iter" % ((time.time() - t0) * 1000 / int(os.environ.get("ITERS", "30"))), flush=True)
