"""N>1 host logic on CPU: owner-major layout, reduce-scatter of mean gradients to
the owners and all-gather of owner results, with world_size 2 and 3 over gloo.

Mirrors the reference's semantics (distsim.py:259-265 mean of local grads;
distsim.py:333-336 owner result broadcast to all)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_15143_b200.exchange import OwnerMajorExchange, OwnerMajorLayout
from paper_2206_15143_b200.partition import balanced_partition, round_robin_partition

SHAPES = [(4, 7), (3, 5), (6, 2), (2, 9), (5, 5)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_grad(rank, i):
    g = torch.Generator().manual_seed(1000 * rank + i)
    return torch.randn(*SHAPES[i], generator=g)


BUCKETS = [[4, 3], [2], [1, 0]]  # backward order, as DPKFAC._grad_buckets cuts them


def _worker(rank, world, port, assign_kind, q, bucketed=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = len(SHAPES)
        if assign_kind == "rr":
            assignment = round_robin_partition(n, world)
        else:
            assignment = balanced_partition([r * c for r, c in SHAPES], world)
        layout = OwnerMajorLayout(assignment, [r * c for r, c in SHAPES], align=4,
                                  buckets=BUCKETS if bucketed else None)
        x = OwnerMajorExchange(layout, rank, "cpu")
        for i in range(n):  # pack (the CUDA pack kernel's job on the GPU): flat = grad / P
            off = layout.in_offsets[i]
            x.flat[off:off + SHAPES[i][0] * SHAPES[i][1]] = (_local_grad(rank, i) / world).reshape(-1)
        if bucketed:  # one collective per bucket, in backward order (as the hooks issue them)
            for b in range(len(layout.buckets)):
                x.reduce_scatter_bucket(b)
        else:
            x.reduce_scatter()
        for i in assignment[rank]:  # "precondition": owner tags its result with (i+1)
            x.view_out(i, SHAPES[i]).copy_(x.view_in(i, SHAPES[i]) * (i + 1))
        x.all_gather()
        out = {}
        for i in range(n):
            off = layout.offsets[i]
            # numpy, pickled by value: torch tensors would travel as shared-memory handles
            # that die with this process before the parent reads them
            out[i] = x.out_flat[off:off + SHAPES[i][0] * SHAPES[i][1]].view(*SHAPES[i]).numpy().copy()
        q.put((rank, out, layout.padding))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,bucketed", [(2, "rr", False), (3, "rr", False), (2, "balanced", False),
                                                (8, "balanced", False), (8, "rr", False), (2, "rr", True),
                                                (3, "balanced", True)])
def test_owner_major_exchange_gloo(world, kind, bucketed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q, bucketed)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i in range(len(SHAPES)):
        mean = sum(_local_grad(r, i) for r in range(world)) / world
        want = mean * (i + 1)
        for rank, out, pad in results:
            assert torch.allclose(torch.from_numpy(out[i]), want, atol=1e-6), (rank, i)
    # replicas identical after the exchange (reference test_distsim.py:203-214)
    base = results[0][1]
    for _, out, _ in results[1:]:
        for i in range(len(SHAPES)):
            assert (out[i] == base[i]).all()


def test_bucketed_layout_offsets():
    """comm_overlap layout: every bucket's reduce-scatter input region holds rank r's
    layers of that bucket at r * bucket_chunk; the gathered layout is rank-major and
    equals the plain owner-major one when there is a single bucket."""
    n_grad = [r * c for r, c in SHAPES]
    assignment = round_robin_partition(len(SHAPES), 2)
    one = OwnerMajorLayout(assignment, n_grad, align=4)
    assert one.in_offsets == one.offsets and one.buckets == ((0, 1, 2, 3, 4),)
    lay = OwnerMajorLayout(assignment, n_grad, align=4, buckets=BUCKETS, scalar_slot=True)
    assert sum(lay.bucket_chunk) == lay.chunk and lay.total == 2 * lay.chunk
    for i, g in enumerate(n_grad):
        p, b = lay.owner_of(i), lay.bucket_of[i]
        base, c = lay.bucket_base[b], lay.bucket_chunk[b]
        assert 2 * base + p * c <= lay.in_offsets[i] and lay.in_offsets[i] + g <= 2 * base + (p + 1) * c
        assert p * lay.chunk + base <= lay.offsets[i] and lay.offsets[i] + g <= p * lay.chunk + base + c
        assert lay.offsets[i] - p * lay.chunk < lay.slot_offset  # the KL slot is never a layer's float
    with pytest.raises(ValueError):
        OwnerMajorLayout(assignment, n_grad, buckets=[[0, 1], [2, 3]])


def _agree_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2206_15143_b200.exchange import agree_max
        from paper_2206_15143_b200.partition import step_time_partition
        # ragged local batches: rank r sees M = 64 - 8 r samples on every layer
        dims = [(785, 512), (513, 256), (257, 10), (1153, 128), (2305, 64)]
        ms = agree_max([64 - 8 * rank] * len(dims))
        q.put((rank, ms, step_time_partition([(a, b, m) for (a, b), m in zip(dims, ms)], world)))
    finally:
        dist.destroy_process_group()


def test_balanced_partition_agrees_across_ranks_with_ragged_batches_gloo():
    """every rank must build the same partition even when local batch
    shapes differ -- the sample counts are MAX-all-reduced before the balancer."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] == [64] * 5 for r in res)
    assert len({r[2] for r in res}) == 1
