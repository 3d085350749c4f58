"""torchrun --nproc-per-node P scripts/nccl_probe.py: reduce-scatter / all-gather of the
ResNet-50 gradient size (25.5 M floats) in isolation, CUDA-event timed, max over ranks."""
import os, sys
import torch, torch.distributed as dist
dist.init_process_group("nccl")
r, P = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
n = 25_557_032 // P * P + 32 * P
flat = torch.randn(n, device=dev)
chunk = torch.empty(n // P, device=dev)
out = torch.empty(n, device=dev)
for _ in range(5):
    dist.reduce_scatter_tensor(chunk, flat)
    dist.all_gather_into_tensor(out, chunk)
torch.cuda.synchronize(); dist.barrier()
res = {}
for name, fn in (("reduce_scatter", lambda: dist.reduce_scatter_tensor(chunk, flat)),
                 ("all_gather", lambda: dist.all_gather_into_tensor(out, chunk)),
                 ("all_reduce", lambda: dist.all_reduce(flat))):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); dist.barrier()
    a.record()
    for _ in range(20):
        fn()
    b.record(); torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / 20], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res[name] = float(t)
if r == 0:
    gb = n * 4 / 1e9
    for k, v in res.items():
        bus = gb * (P - 1) / P / (v / 1e3) * (2 if k == "all_reduce" else 1)
        print(f"P={P} {k}: {v:.3f} ms for {gb*1e3:.0f} MB (bus {bus:.0f} GB/s) env NCCL_ALGO={os.environ.get('NCCL_ALGO')} NVLS={os.environ.get('NCCL_NVLS_ENABLE')}", flush=True)
dist.destroy_process_group()
