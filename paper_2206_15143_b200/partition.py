"""Layer -> GPU assignment for DP-KFAC.

``round_robin_partition`` is the reference's partition, bit for bit
(kfaclab costmodel.py:66-70, used by distsim.assign_layers_round_robin
distsim.py:86-90); ``validate_partition`` mirrors distsim.py:93-101.

``balanced_partition`` is the flop load balancer:
deterministic longest-processing-time-first over a per-layer cost model of
the second-order work (factor SYRKs + inversion/eigendecomposition +
preconditioning), tie-broken by layer index and then by rank.

``step_time_partition`` (what DPKFAC's assignment="balanced" uses) balances an
estimated B200 step time per rank instead of flops alone: throughput work, the
latency-bound inversion chain of each rank's largest factor, and the owner-major
exchange, whose chunk (and so its NCCL traffic) is the LARGEST rank's gradient
count -- a flop-only LPT pads ResNet-50's exchange by 57% at P=8.  Greedy
placement in decreasing size, then deterministic move/swap improvement.
"""

from __future__ import annotations

import os

from typing import Sequence

from .errors import ArgumentError


def round_robin_partition(n_layers: int, workers: int) -> tuple[tuple[int, ...], ...]:
    """Worker p owns layers p, p+P, p+2P, ... (reference costmodel.py:66-70)."""
    if n_layers < 0 or workers < 1:
        raise ArgumentError("need n_items >= 0 and n_workers >= 1")
    return tuple(tuple(range(p, n_layers, workers)) for p in range(workers))


def assign_layers_round_robin(n_layers: int, workers: int) -> tuple[tuple[int, ...], ...]:
    """reference distsim.py:86-90."""
    if n_layers < 1:
        raise ArgumentError("need at least one layer")
    return round_robin_partition(n_layers, workers)


def validate_partition(assignment: Sequence[Sequence[int]], n_layers: int) -> None:
    """Every layer owned by exactly one worker (reference distsim.py:93-101)."""
    seen: set[int] = set()
    for part in assignment:
        for i in part:
            if i in seen:
                raise ArgumentError(f"layer {i} assigned to more than one worker")
            seen.add(i)
    if seen != set(range(n_layers)):
        raise ArgumentError(f"assignment does not cover layers 0..{n_layers - 1} exactly")


def layer_cost(d_in: int, d_out: int, m: int, inv_type: str = "inverse") -> float:
    """Second-order work of one layer in flops: unique-output SYRKs for A and G,
    n^3 (Cholesky-grade inverse) or ~9 n^3 (eigen) per factor, and the two-sided
    preconditioning products."""
    syrk = (d_in * (d_in + 1) + d_out * (d_out + 1)) * float(m)
    cube = float(d_in) ** 3 + float(d_out) ** 3
    decomp = cube if inv_type == "inverse" else 9.0 * cube
    pre = 2.0 * (d_out * d_out * d_in + d_out * d_in * d_in) * (1 if inv_type == "inverse" else 2)
    return syrk + decomp + pre


def balanced_partition(costs: Sequence[float], workers: int) -> tuple[tuple[int, ...], ...]:
    """Deterministic LPT: layers by descending cost (ties: lower index first) go to
    the currently least-loaded worker (ties: lower rank).  Each worker's layers
    are returned in ascending order, as the reference iterates them (distsim.py:312)."""
    if workers < 1:
        raise ArgumentError("need n_workers >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    load = [0.0] * workers
    parts: list[list[int]] = [[] for _ in range(workers)]
    for i in order:
        p = min(range(workers), key=lambda r: (load[r], r))
        parts[p].append(i)
        load[p] += float(costs[i])
    return tuple(tuple(sorted(p)) for p in parts)


def imbalance(costs: Sequence[float], assignment: Sequence[Sequence[int]]) -> float:
    """max worker load / mean worker load."""
    loads = [sum(costs[i] for i in part) for part in assignment]
    mean = sum(loads) / len(loads)
    return max(loads) / mean if mean > 0 else 1.0


# B200 rates of the stages, measured: factor SYRKs ~500 TF/s
# effective (kind::f16 conv patches after the MMA issue-loop fix; 340 before),
# 3xTF32 inversion rounds ~100 TF/s, preconditioning ~110 TF/s; the blocked SPD
# inversion of an n > 128 factor is a dependent chain of ~0.7 us per row (4608: ~3 ms);
# NCCL reduce-scatter + all-gather at ~450 GB/s bus bandwidth.  Re-fit at the end of
# round 2 by measuring the step (scripts/gpu_runs/r2_balfit*.sh): N=4 4.06 -> 3.79 ms,
# N=2 4.90 -> 4.92 ms.
RATE_SYRK = 500e12
RATE_INV = 100e12
RATE_PRE = 110e12
CHAIN_S_PER_ROW = 0.7e-6
BUS_BYTES_PER_S = 450e9


def _rate(name: str, default: float) -> float:  # DPK_BAL_<NAME>: model re-fit experiments
    v = os.environ.get("DPK_BAL_" + name)
    return float(v) if v else default


def layer_time(d_in: int, d_out: int, m: int, inv_type: str = "inverse") -> tuple[float, float]:
    """(throughput seconds, latency-chain seconds) of one layer's second-order work."""
    syrk = (d_in * (d_in + 1) + d_out * (d_out + 1)) * float(m)
    cube = float(d_in) ** 3 + float(d_out) ** 3
    inv = (2.0 / 3.0) * cube if inv_type == "inverse" else 9.0 * cube
    pre = 2.0 * (d_out * d_out * d_in + d_out * d_in * d_in) * (1 if inv_type == "inverse" else 2)
    work = syrk / _rate("SYRK", RATE_SYRK) + inv / _rate("INV", RATE_INV) + pre / _rate("PRE", RATE_PRE)
    big = max(d_in, d_out)
    chain = _rate("CHAIN", CHAIN_S_PER_ROW) * big if (big > 128 and inv_type == "inverse") else 0.0
    return work, chain


def _step_time(loads, chains, grads, workers):
    comp = max(max(w, c) for w, c in zip(loads, chains))
    comm = 2.0 * (workers - 1) * max(grads) * 4.0 / BUS_BYTES_PER_S if workers > 1 else 0.0
    return comp + comm


def step_time_partition(layers: Sequence[tuple], workers: int, inv_type: str = "inverse",
                        max_rounds: int = 200) -> tuple[tuple[int, ...], ...]:
    """layers: (d_in, d_out, m) per layer.  Deterministic: same input -> same partition."""
    if workers < 1:
        raise ArgumentError("need n_workers >= 1")
    n = len(layers)
    t = [layer_time(a, b, m, inv_type) for a, b, m in layers]
    ng = [a * b for a, b, _ in layers]
    owner = [0] * n
    loads, chains, grads = [0.0] * workers, [0.0] * workers, [0] * workers
    parts: list[list[int]] = [[] for _ in range(workers)]
    order = sorted(range(n), key=lambda i: (-max(t[i][0], t[i][1]), -ng[i], i))
    for i in order:
        best, best_r = None, 0
        for r in range(workers):
            loads[r] += t[i][0]
            grads[r] += ng[i]
            oc = chains[r]
            chains[r] = max(oc, t[i][1])
            v = (_step_time(loads, chains, grads, workers), loads[r] + grads[r] * 1e-12, r)
            loads[r] -= t[i][0]
            grads[r] -= ng[i]
            chains[r] = oc
            if best is None or v < best:
                best, best_r = v, r
        owner[i] = best_r
        parts[best_r].append(i)
        loads[best_r] += t[i][0]
        grads[best_r] += ng[i]
        chains[best_r] = max(chains[best_r], t[i][1])

    members = [set(p) for p in parts]

    def chain_of(r):
        return max([t[i][1] for i in members[r]] or [0.0])

    def try_assign(moves):
        """Apply [(layer, new rank)], return the step time, undo."""
        touched = {owner[i] for i, _ in moves} | {r for _, r in moves}
        saved = {r: (loads[r], grads[r], chains[r]) for r in touched}
        old = [(i, owner[i]) for i, _ in moves]
        for i, r in moves:
            r0 = owner[i]
            loads[r0] -= t[i][0]
            grads[r0] -= ng[i]
            members[r0].discard(i)
            loads[r] += t[i][0]
            grads[r] += ng[i]
            members[r].add(i)
            owner[i] = r
        for r in touched:
            chains[r] = chain_of(r)
        v = _step_time(loads, chains, grads, workers)
        for i, r0 in reversed(old):
            r = owner[i]
            members[r].discard(i)
            members[r0].add(i)
            owner[i] = r0
        for r, (a, b, c) in saved.items():
            loads[r], grads[r], chains[r] = a, b, c
        return v

    def commit(moves):
        for i, r in moves:
            r0 = owner[i]
            loads[r0] -= t[i][0]
            grads[r0] -= ng[i]
            members[r0].discard(i)
            loads[r] += t[i][0]
            grads[r] += ng[i]
            members[r].add(i)
            owner[i] = r
        for r in range(workers):
            chains[r] = chain_of(r)

    cur = _step_time(loads, chains, grads, workers)
    for _ in range(max_rounds):
        # only the bottleneck ranks can lower the step time: the slowest compute
        # rank and the rank with the most gradient elements (the chunk size)
        slow = max(range(workers), key=lambda r: (max(loads[r], chains[r]), -r))
        fat = max(range(workers), key=lambda r: (grads[r], -r))
        best = None
        srcs = sorted({slow, fat})
        for src in srcs:  # best single move out of a bottleneck rank
            for i in sorted(members[src]):
                for r in range(workers):
                    if r != src:
                        v = try_assign([(i, r)])
                        if v < cur * (1 - 1e-9) and (best is None or v < best[0]):
                            best = (v, [(i, r)])
        if best is None:  # else the best swap with another rank
            for src in srcs:
                for i in sorted(members[src]):
                    for r in range(workers):
                        if r == src:
                            continue
                        for j in sorted(members[r]):
                            v = try_assign([(i, r), (j, src)])
                            if v < cur * (1 - 1e-9) and (best is None or v < best[0]):
                                best = (v, [(i, r), (j, src)])
        if best is None:
            break
        commit(best[1])
        cur = best[0]
    out = [[] for _ in range(workers)]
    for i in range(n):
        out[owner[i]].append(i)
    return tuple(tuple(p) for p in out)


def partition_report(layers: Sequence[tuple], assignment, inv_type: str = "inverse") -> dict:
    """Estimated step time, flop imbalance and owner-major padding of a partition."""
    P = len(assignment)
    t = [layer_time(a, b, m, inv_type) for a, b, m in layers]
    ng = [a * b for a, b, _ in layers]
    loads = [sum(t[i][0] for i in p) for p in assignment]
    chains = [max([t[i][1] for i in p] or [0.0]) for p in assignment]
    grads = [sum(ng[i] for i in p) for p in assignment]
    pad = 1.0 - sum(ng) / (P * max(grads)) if max(grads) else 0.0
    return {"est_ms": 1e3 * _step_time(loads, chains, grads, P), "padding": pad,
            "work_imbalance": max(loads) / (sum(loads) / P), "max_chain_ms": 1e3 * max(chains)}
