"""Profiling driver: ResNet-50 captures resident, a few warm-up DP-KFAC steps, then
exactly ``--profiled`` steps inside cudaProfilerStart/Stop (use ncu
--profile-from-start off).  Prints per-stage CUDA-event times of the profiled steps."""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import torch.nn.functional as F

import bench_models as BM
from paper_2206_15143_b200 import DPKFAC

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="resnet50")
ap.add_argument("--inv-type", default="inverse")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--profiled", type=int, default=1)
ap.add_argument("--precision", default="tf32")
ap.add_argument("--nchw", action="store_true", help="keep the model NCHW (default: channels_last)")
args = ap.parse_args()

dev = torch.device("cuda", 0)
ctor, batch, shape, classes = BM.WORKLOADS[args.model]
torch.manual_seed(0)
model = ctor().to(dev)
mf = torch.contiguous_format if args.nchw else torch.channels_last
if len(shape) == 3:
    model = model.to(memory_format=mf)
kf = DPKFAC(model, gamma=0.002, xi=0.95, inv_type=args.inv_type, precision=args.precision,
            check_numerics="deferred")
x = torch.randn(batch, *shape, device=dev)
if len(shape) == 3:
    x = x.contiguous(memory_format=mf)
y = torch.randint(0, classes, (batch,), device=dev)
F.cross_entropy(model(x), y).backward()
kf.step()
model.zero_grad(set_to_none=False)
F.cross_entropy(model(x), y).backward()
caps = {ly.index: (ly.a_in, ly.g_out, ly.batch) for ly in kf.owned}


def restore():
    for ly in kf.owned:
        ly.a_in, ly.g_out, ly.batch = caps[ly.index]


for _ in range(args.warmup):
    restore()
    kf.step()
torch.cuda.synchronize()
kf.enable_stage_timing(True)
torch.cuda.cudart().cudaProfilerStart()
for _ in range(args.profiled):
    restore()
    kf.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print({k: round(v / args.profiled, 3) for k, v in kf.stage_ms().items()})
kf.check()
