"""Owner-major gradient exchange of DP-KFAC over torch.distributed (NCCL on B200).

Replaces the reference's per-layer averaging all-reduce (distsim._aggregate_grads,
distsim.py:259-265) and the per-layer broadcast of preconditioned gradients from
each owner (distsim.py:333-336) with exactly two collectives per step:

  flat  = [ rank 0's layers | pad | rank 1's layers | pad | ... ]   (each region = ``chunk`` floats)
  reduce_scatter(flat / P)  ->  chunk_in  = mean gradients of MY layers only
  (owner preconditions chunk_in -> chunk_out)
  all_gather(chunk_out)     ->  out_flat  = every layer's preconditioned gradient

Per rank this moves 2 (P-1)/P * P*chunk floats, no Kronecker factor ever moves
(SPEC: DP-KFAC FactorComm = 0).  The layout logic is device-agnostic so it is
exercised by the CPU gloo tests as well.
"""

from __future__ import annotations

from typing import Optional, Sequence

import torch
import torch.distributed as dist


class OwnerMajorLayout:
    """``scalar_slot``: reserve the last float of every rank's chunk for one per-rank
    scalar that rides the all-gather (the KL-clip partial dot): ``slot_offset``
    inside a chunk, ``chunk`` apart in the gathered buffer.

    ``buckets`` (layer index lists covering every layer once; default one bucket):
    the reduce-scatter is split into one collective per bucket so it can run as
    soon as the backward pass has produced that bucket's gradients.
    A rank's chunk is then the concatenation of its per-bucket parts, each padded
    to the bucket's largest part (``bucket_chunk[b]`` floats at ``bucket_base[b]``):

      pack buffer  flat     = [bucket 0: r0 | r1 | ... ][bucket 1: r0 | r1 | ... ] ...
      RS of bucket b        : flat[P*base_b : P*(base_b + chunk_b)] -> chunk_in[base_b : base_b + chunk_b]
      gathered     out_flat = [rank 0: b0 | b1 | ... ][rank 1: b0 | b1 | ... ] ...

    so layers are packed at ``in_offsets`` and unpacked from ``offsets``; with one
    bucket the two coincide and the layout is the plain owner-major one."""

    def __init__(self, assignment: Sequence[Sequence[int]], n_grad: Sequence[int], align: int = 32,
                 scalar_slot: bool = False, buckets: Optional[Sequence[Sequence[int]]] = None):
        self.assignment = tuple(tuple(p) for p in assignment)
        self.world = len(self.assignment)
        self.n_grad = list(n_grad)
        if buckets is None:
            buckets = [sorted(i for part in self.assignment for i in part)]
        self.buckets = tuple(tuple(int(i) for i in b) for b in buckets)
        seen = sorted(i for b in self.buckets for i in b)
        if seen != sorted(i for part in self.assignment for i in part):
            raise ValueError("buckets must cover every assigned layer exactly once")
        bucket_of = {i: k for k, b in enumerate(self.buckets) for i in b}
        self.bucket_of = bucket_of
        nb = len(self.buckets)
        # per (bucket, rank) part sizes; the KL slot rides at the end of the last bucket
        sizes = [[0] * self.world for _ in range(nb)]
        for p, part in enumerate(self.assignment):
            for i in part:
                sizes[bucket_of[i]][p] += self.n_grad[i]
        self.bucket_chunk, self.bucket_base = [], []
        base = 0
        for k in range(nb):
            c = max(max(sizes[k]) if sizes[k] else 0, 1 if nb == 1 else 0) + (1 if scalar_slot and k == nb - 1 else 0)
            c = (c + align - 1) // align * align
            self.bucket_base.append(base)
            self.bucket_chunk.append(c)
            base += c
        self.chunk = max(base, align)
        if self.chunk > base:  # (only an empty single bucket) keep the padding in the last bucket
            self.bucket_chunk[-1] += self.chunk - base
        self.slot_offset = self.chunk - 1 if scalar_slot else None
        self.offsets = {}      # gathered (rank-major) layout: unpack / preconditioned output
        self.in_offsets = {}   # pack (bucket-major) layout: the reduce-scatter input
        self._local = {}
        for p, part in enumerate(self.assignment):
            fill = list(self.bucket_base)
            for i in part:
                k = bucket_of[i]
                loc = fill[k]
                fill[k] += self.n_grad[i]
                self._local[i] = loc
                self.offsets[i] = p * self.chunk + loc
                self.in_offsets[i] = (self.world * self.bucket_base[k] + p * self.bucket_chunk[k] +
                                      loc - self.bucket_base[k])
        self.total = self.world * self.chunk
        # elements that travel but carry no gradient (equal-chunk padding for NCCL RS/AG)
        self.padding = self.total - sum(self.n_grad)

    def owner_of(self, layer: int) -> int:
        for p, part in enumerate(self.assignment):
            if layer in part:
                return p
        raise KeyError(layer)

    def local_offset(self, layer: int, rank: int) -> int:
        """Offset of an owned layer inside that rank's chunk."""
        return self._local[layer]


class OwnerMajorExchange:
    """Buffers + the two collectives.  For world == 1 no collective is issued."""

    def __init__(self, layout: OwnerMajorLayout, rank: int, device, group=None):
        self.layout = layout
        self.rank = rank
        self.group = group
        P, c = layout.world, layout.chunk
        self.flat = torch.zeros(P * c, device=device)
        if P == 1:
            self.chunk_in = self.flat
            self.chunk_out = torch.zeros(c, device=device)
            self.out_flat = self.chunk_out
        else:
            self.chunk_in = torch.zeros(c, device=device)
            self.chunk_out = torch.zeros(c, device=device)
            self.out_flat = torch.zeros(P * c, device=device)
        self.chunk_tmp = torch.zeros(c, device=device)
        self._peer_ptrs = None  # enable_peer_gather(): every rank's chunk_out, IPC-mapped

    def enable_peer_gather(self) -> bool:
        """Replace the closing NCCL all-gather by one copy kernel that reads every
        rank's chunk_out in place over NVLink (dpk_peer_gather): the chunk buffers are
        IPC-mapped once here.  Single node only; every rank takes the same decision
        (it returns False, and the NCCL collective stays, unless all ranks can)."""
        import ctypes as C
        import socket
        from . import _lib as L
        from .ops import lib
        P = self.layout.world
        if P == 1 or P > 8:
            return False
        co = self.chunk_out
        buf, off = C.create_string_buffer(64), C.c_int64(0)
        # e.g. expandable segments (no cudaMalloc segment behind the block): NCCL stays
        ok = lib().dpk_ipc_export(co.data_ptr(), co.device.index, buf, C.byref(off)) == L.DPK_OK
        handle, off = buf.raw, int(off.value)
        mine = (socket.gethostname(), handle, off, ok)
        objs = [None] * P
        dist.all_gather_object(objs, mine, group=self.group)
        if not all(o[3] for o in objs) or len({o[0] for o in objs}) != 1:
            return False
        ptrs = []
        for r, (_, h, o, _) in enumerate(objs):
            if r == self.rank:
                ptrs.append(co.data_ptr())
                continue
            base = C.c_void_p()
            L.check(lib().dpk_ipc_open(h, co.device.index, C.byref(base)), "dpk_ipc_open")
            ptrs.append(base.value + o)
        self._peer_ptrs = (C.c_void_p * P)(*ptrs)
        self._ready = torch.zeros(1, device=co.device)
        return True

    def reduce_scatter(self):
        """flat must already hold grad / P (pack scale); SUM then equals the mean."""
        for b in range(len(self.layout.buckets)):
            self.reduce_scatter_bucket(b)

    def reduce_scatter_bucket(self, b: int):
        """The reduce-scatter of one gradient bucket (its region of flat must be packed)."""
        if self.layout.world > 1:
            L_ = self.layout
            base, c, P = L_.bucket_base[b], L_.bucket_chunk[b], L_.world
            dist.reduce_scatter_tensor(self.chunk_in[base:base + c], self.flat[P * base:P * (base + c)],
                                       op=dist.ReduceOp.SUM, group=self.group)

    def all_gather(self):
        if self.layout.world > 1:
            if self._peer_ptrs is not None:
                # stream-ordered readiness: this tiny all-reduce completes only once
                # every rank has reached it, i.e. finished writing its chunk_out; the
                # next step's reduce-scatter orders the reads before any rewrite
                dist.all_reduce(self._ready, group=self.group)
                from .ops import peer_gather
                peer_gather(self.out_flat, self._peer_ptrs, self.layout.world, self.layout.chunk)
                return
            dist.all_gather_into_tensor(self.out_flat, self.chunk_out, group=self.group)

    def view_in(self, layer: int, shape):
        off = self.layout.local_offset(layer, self.rank)
        n = shape[0] * shape[1]
        return self.chunk_in[off:off + n].view(*shape)

    def view_out(self, layer: int, shape):
        off = self.layout.local_offset(layer, self.rank)
        n = shape[0] * shape[1]
        return self.chunk_out[off:off + n].view(*shape)

    def view_tmp(self, layer: int, shape):
        off = self.layout.local_offset(layer, self.rank)
        n = shape[0] * shape[1]
        return self.chunk_tmp[off:off + n].view(*shape)


def agree_max(values, group=None, device="cpu"):
    """Element-wise MAX of a per-rank integer list over the group (identity when
    not distributed): every rank then feeds the same numbers to the deterministic
    balancer, so all ranks build the same owner-major layout."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return [int(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [int(v) for v in t.tolist()]
