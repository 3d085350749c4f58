"""Layer -> GPU assignment for DP-KFAC.

``round_robin_partition`` is the reference's partition, bit for bit
(kfaclab costmodel.py:66-70, used by distsim.assign_layers_round_robin
distsim.py:86-90); ``validate_partition`` mirrors distsim.py:93-101.

``balanced_partition`` is the opt-in load balancer:
deterministic longest-processing-time-first over a per-layer cost model of
the second-order work (factor SYRKs + inversion/eigendecomposition +
preconditioning), tie-broken by layer index and then by rank.
"""

from __future__ import annotations

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
