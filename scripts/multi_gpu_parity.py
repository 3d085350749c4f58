"""torchrun --nproc-per-node P scripts/multi_gpu_parity.py: DP-KFAC and the MPD-KFAC
comparators over NCCL vs the oracle's P-worker simulation (distsim semantics), on an
MLP whose global batch is sharded contiguously (distsim.shard_batch 'disjoint')."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import torch.distributed as dist
import torch.nn.functional as F

from oracle import kfac_ref as K  # the checker
from oracle import mlp_ref as MLP
from paper_2206_15143_b200 import DPKFAC


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def main():
    dist.init_process_group("nccl")
    rank, P = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    spec = MLP.MlpSpec((20, 16, 12, 5), "relu", "softmax_cross_entropy", True)
    B = 8 * P
    bad = []
    for algorithm, inv in [("dp_kfac", "inverse"), ("dp_kfac", "eigen"), ("mpd_kfac_co", "inverse"),
                           ("mpd_kfac_mo", "inverse"), ("mpd_kfac_co", "eigen"), ("dp_kfac:balanced", "inverse"),
                           ("dp_kfac:round_robin+overlap", "inverse"), ("dp_kfac:balanced+overlap", "eigen"),
                           ("dp_kfac:balanced+peer", "inverse"), ("dp_kfac:round_robin+peer", "eigen")]:
        alg, _, asg = algorithm.partition(":")
        # +overlap: bucketed reduce-scatter from the backward hooks, one layer per bucket;
        # +peer: the closing all-gather as the NVLink peer-copy kernel
        asg, _, ov = asg.partition("+")
        h = K.Hyper(gamma=0.05, xi=0.9, inv_type=inv, f_freq=1, k_freq=2)
        cl = (MLP.build_cluster if alg == "dp_kfac" else MLP.build_mpd_cluster)(spec, P, seed=5)
        mods = []
        for i, w in enumerate(cl.weights):
            lin = torch.nn.Linear(w.shape[1] - 1, w.shape[0])
            with torch.no_grad():
                lin.weight.copy_(torch.from_numpy(w[:, :-1]))
                lin.bias.copy_(torch.from_numpy(w[:, -1]))
            mods += [lin, torch.nn.ReLU()]
        model = torch.nn.Sequential(*mods[:-1]).to(dev)
        lins = [m for m in model if isinstance(m, torch.nn.Linear)]
        kf = DPKFAC(model, gamma=0.05, xi=0.9, inv_type=inv, k_freq=2, precision="3xtf32", algorithm=alg,
                    assignment=asg or "round_robin", comm_overlap=ov == "overlap", bucket_mb=1e-4,
                    peer_gather=ov == "peer")
        opt = torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9)
        rng = np.random.default_rng(91)
        for t in range(4):
            x, y = rng.standard_normal((20, B)), rng.integers(0, 5, size=B)
            if asg == "balanced" and t == 0:
                pass  # the oracle cluster must use the same partition: set after the first capture
            shards = MLP.shard(x, y, P)
            xs, ys = shards[rank]
            opt.zero_grad()
            F.cross_entropy(model(torch.from_numpy(xs.T.copy()).float().to(dev)),
                            torch.from_numpy(ys).to(dev)).backward()
            if ov == "overlap" and t > 0 and len(kf._bucket_ev) != len(kf.layout.buckets):
                bad.append((algorithm, inv, t, "hooks did not launch every bucket"))
            kf.step()
            if ov == "peer" and t == 0 and kf.xchg._peer_ptrs is None:
                bad.append((algorithm, inv, "peer gather not enabled"))
            if asg == "balanced" and t == 0:
                cl = MLP.build_cluster(spec, P, seed=5, assignment=kf.assignment)
            if alg == "dp_kfac":
                _, pre = MLP.dp_kfac_step(cl, shards, h, 0.1, 0.9, t)
            else:
                _, pre = MLP.mpd_kfac_step(cl, shards, h, 0.1, 0.9, t, alg[-2:])
            for i, lin in enumerate(lins):
                got = torch.cat([lin.weight.grad, lin.bias.grad[:, None]], 1).double().cpu().numpy()
                e = rel(got, pre[i])
                if not e <= 1e-3:
                    bad.append((algorithm, inv, t, i, e))
            opt.step()
        for i, lin in enumerate(lins):
            got = torch.cat([lin.weight, lin.bias[:, None]], 1).detach().double().cpu().numpy()
            if not rel(got, cl.weights[i]) <= 1e-4:
                bad.append((algorithm, inv, "weights", i, rel(got, cl.weights[i])))
        kf.remove_hooks()
    # KL-clip over NCCL: every rank's partial <pre, grad> rides the all-gather (one slot per
    # owner chunk); the unpack applies nu = min(1, sqrt(kl / |lr^2 sum <pre, grad>|))
    for inv, peer in (("inverse", False), ("eigen", False), ("inverse", True)):
        h = K.Hyper(gamma=0.05, xi=0.9, inv_type=inv, f_freq=1, k_freq=1)
        cl = MLP.build_cluster(spec, P, seed=7)
        mods = []
        for i, w in enumerate(cl.weights):
            lin = torch.nn.Linear(w.shape[1] - 1, w.shape[0])
            with torch.no_grad():
                lin.weight.copy_(torch.from_numpy(w[:, :-1]))
                lin.bias.copy_(torch.from_numpy(w[:, -1]))
            mods += [lin, torch.nn.ReLU()]
        model = torch.nn.Sequential(*mods[:-1]).to(dev)
        lins = [m for m in model if isinstance(m, torch.nn.Linear)]
        lr, kl = 0.1, 1e-5
        kf = DPKFAC(model, gamma=0.05, xi=0.9, inv_type=inv, precision="3xtf32", kl_clip=kl, lr=lr,
                    assignment="balanced", peer_gather=peer)
        rng = np.random.default_rng(17)
        x, y = rng.standard_normal((20, B)), rng.integers(0, 5, size=B)
        shards = MLP.shard(x, y, P)
        xs, ys = shards[rank]
        F.cross_entropy(model(torch.from_numpy(xs.T.copy()).float().to(dev)), torch.from_numpy(ys).to(dev)).backward()
        kf.step()
        cl = MLP.build_cluster(spec, P, seed=7, assignment=kf.assignment)
        _, pre = MLP.dp_kfac_step(cl, shards, h, lr, 0.9, 0)
        loc = [MLP.forward_backward(spec, MLP.init_weights(spec, 7), xx, yy)[3] for xx, yy in shards]
        agg = [MLP.tree_mean([loc[p][i] for p in range(P)]) for i in range(len(lins))]
        vg = sum(float((pre[i] * agg[i]).sum()) for i in range(len(lins))) * lr * lr
        nu = min(1.0, (kl / abs(vg)) ** 0.5)
        if not nu < 1.0:
            bad.append(("kl_clip inactive", inv, nu))
        for i, lin in enumerate(lins):
            got = torch.cat([lin.weight.grad, lin.bias.grad[:, None]], 1).double().cpu().numpy()
            e = rel(got, nu * pre[i])
            if not e <= 1e-3:
                bad.append(("kl_clip", inv, i, e, nu))
        kf.remove_hooks()
    # non-preconditioned parameters (batch norm) are averaged over ranks, unpreconditioned
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Linear(20, 16), torch.nn.BatchNorm1d(16), torch.nn.ReLU(),
                              torch.nn.Linear(16, 5)).to(dev)
    kf = DPKFAC(net, gamma=0.05, xi=0.9, inv_type="inverse", precision="3xtf32")
    gen = torch.Generator().manual_seed(100 + rank)
    xb = torch.randn(8, 20, generator=gen).to(dev)
    yb = torch.randint(0, 5, (8,), generator=gen).to(dev)
    F.cross_entropy(net(xb), yb).backward()
    bn = net[1]
    local = torch.cat([bn.weight.grad, bn.bias.grad]).clone()
    allg = [torch.empty_like(local) for _ in range(P)]
    dist.all_gather(allg, local)
    kf.step()
    mean = sum(allg) / P
    got = torch.cat([bn.weight.grad, bn.bias.grad])
    if not torch.allclose(got, mean, rtol=1e-6, atol=1e-7):
        bad.append(("batchnorm mean", float((got - mean).abs().max())))
    kf.remove_hooks()
    flag = torch.tensor([len(bad)], device=dev)
    dist.all_reduce(flag)
    if rank == 0:
        print("PARITY OK" if int(flag) == 0 else f"PARITY FAILED {bad}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(flag) == 0 else 1)


if __name__ == "__main__":
    main()
