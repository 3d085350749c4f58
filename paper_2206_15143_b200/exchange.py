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

from typing import Sequence

import torch
import torch.distributed as dist


class OwnerMajorLayout:
    """``scalar_slot``: reserve the last float of every rank's chunk for one per-rank
    scalar that rides the all-gather (the KL-clip partial dot): ``slot_offset``
    inside a chunk, ``chunk`` apart in the gathered buffer."""

    def __init__(self, assignment: Sequence[Sequence[int]], n_grad: Sequence[int], align: int = 32,
                 scalar_slot: bool = False):
        self.assignment = tuple(tuple(p) for p in assignment)
        self.world = len(self.assignment)
        self.n_grad = list(n_grad)
        sizes = [sum(self.n_grad[i] for i in part) for part in self.assignment]
        chunk = max(max(sizes) if sizes else 0, 1) + (1 if scalar_slot else 0)
        self.chunk = (chunk + align - 1) // align * align
        self.slot_offset = self.chunk - 1 if scalar_slot else None
        self.offsets = {}
        for p, part in enumerate(self.assignment):
            off = p * self.chunk
            for i in part:
                self.offsets[i] = off
                off += self.n_grad[i]
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
        return self.offsets[layer] - rank * self.chunk


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

    def reduce_scatter(self):
        """flat must already hold grad / P (pack scale); SUM then equals the mean."""
        if self.layout.world > 1:
            dist.reduce_scatter_tensor(self.chunk_in, self.flat, op=dist.ReduceOp.SUM, group=self.group)

    def all_gather(self):
        if self.layout.world > 1:
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
