"""float64 restatement of the reference MLP + simulated DP-KFAC step (TEST INFRASTRUCTURE ONLY).

This is the end-to-end oracle for BASELINE config 1 (784-512-256-10 MLP,
batch 64): it reproduces ``kfaclab.distsim.dp_kfac_step`` (distsim.py:289-338)
on the reference fully-connected network (model.py:125-300), so the GPU
``DPKFAC`` optimizer can be checked over several iterations and P workers.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .kfac_ref import (Hyper, LayerState, OracleArgumentError, OracleError, kfac_layer_step,
                       round_robin_partition, validate_partition)


@dataclass(frozen=True)
class MlpSpec:
    """reference model.py:53-82 (NetworkSpec) restricted to what the path needs."""

    dims: tuple
    activation: str = "relu"
    loss: str = "softmax_cross_entropy"
    bias: bool = True  # "homogeneous" bias mode

    @property
    def depth(self):
        return len(self.dims) - 1

    def weight_shape(self, i):
        return self.dims[i + 1], self.dims[i] + (1 if self.bias else 0)


def init_weights(spec: MlpSpec, seed: int):
    """Uniform on +-sqrt(6/(rows+cols)), one rng stream in layer order (model.py:125-137)."""
    rng = np.random.default_rng(seed)
    ws = []
    for i in range(spec.depth):
        r, c = spec.weight_shape(i)
        lim = np.sqrt(6.0 / (r + c))
        ws.append(rng.uniform(-lim, lim, size=(r, c)))
    return ws


def _act(kind, s):
    if kind == "relu":
        return np.maximum(s, 0.0)
    if kind == "tanh":
        return np.tanh(s)
    return s


def _act_deriv(kind, s):
    if kind == "relu":
        return (s > 0.0).astype(np.float64)
    if kind == "tanh":
        t = np.tanh(s)
        return 1.0 - t * t
    return np.ones_like(s)


def _aug(spec, a):
    return np.vstack([a, np.ones((1, a.shape[1]))]) if spec.bias else a


def forward_backward(spec: MlpSpec, ws, x, y):
    """Mean loss, per-layer captures and mean-loss gradients (model.py:207-252).

    Returns (loss, inputs[i] = augmented layer input d_in x B,
    preact_grads[i] = per-sample pre-activation grads d_out x B (not / B),
    grads[i] = (1/B) g a^T).
    """
    B = x.shape[1]
    inputs, pre = [], []
    a = x
    for i, w in enumerate(ws):
        ai = _aug(spec, a)
        inputs.append(ai)
        s = w @ ai
        pre.append(s)
        a = _act(spec.activation, s) if i < spec.depth - 1 else s
    if spec.loss == "softmax_cross_entropy":
        z = a - a.max(axis=0, keepdims=True)
        lse = np.log(np.exp(z).sum(axis=0))
        loss = float(np.mean(lse - z[y, np.arange(B)]))
        p = np.exp(z) / np.exp(z).sum(axis=0, keepdims=True)
        g = p.copy()
        g[y, np.arange(B)] -= 1.0
    else:
        d = a - y
        loss = float(np.mean(0.5 * (d * d).sum(axis=0)))
        g = d
    grads = [None] * spec.depth
    pgrads = [None] * spec.depth
    for i in range(spec.depth - 1, -1, -1):
        pgrads[i] = g
        grads[i] = g @ inputs[i].T / B
        if i > 0:
            core = ws[i][:, :-1] if spec.bias else ws[i]
            g = _act_deriv(spec.activation, pre[i - 1]) * (core.T @ g)
    return loss, inputs, pgrads, grads


def tree_mean(arrs):
    """Fixed index-ordered pairwise tree sum, then / P (distsim.py:166-196)."""
    level = [a.copy() for a in arrs]
    while len(level) > 1:
        nxt = [level[i] + level[i + 1] for i in range(0, len(level) - 1, 2)]
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    return level[0] / len(arrs)


@dataclass
class Cluster:
    """Replicated weights/momenta plus per-owner factor states (distsim.py:135-159)."""

    spec: MlpSpec
    workers: int
    assignment: tuple
    weights: list
    momenta: list
    states: list = field(default_factory=list)  # states[p][i] for owned i


def build_cluster(spec: MlpSpec, workers: int, seed: int, assignment=None) -> Cluster:
    ws = init_weights(spec, seed)
    if assignment is None:
        if spec.depth < 1:
            raise OracleArgumentError("need at least one layer")
        assignment = round_robin_partition(spec.depth, workers)
    validate_partition(assignment, spec.depth)
    return Cluster(spec, workers, tuple(tuple(p) for p in assignment),
                   [w.copy() for w in ws], [np.zeros_like(w) for w in ws],
                   [{i: LayerState() for i in assignment[p]} for p in range(workers)])


def shard(x, y, workers):
    """Contiguous equal column slices (distsim.py:214-233, 'disjoint')."""
    B = x.shape[1]
    if B % workers:
        raise OracleArgumentError(f"batch of {B} samples does not divide across {workers} workers")
    s = B // workers
    return [(x[:, p * s:(p + 1) * s], y[p * s:(p + 1) * s]) for p in range(workers)]


def dp_kfac_step(cl: Cluster, shards, h: Hyper, lr: float, mu: float, t: int):
    """One DP-KFAC iteration (distsim.py:289-338): local captures, mean grads,
    owner preconditions its layers in ascending order, broadcast, heavy-ball."""
    losses, caps, locgrads = [], [], []
    for x, y in shards:
        loss, ins, pgs, gs = forward_backward(cl.spec, cl.weights, x, y)
        losses.append(loss)
        caps.append((ins, pgs))
        locgrads.append(gs)
    agg = [tree_mean([locgrads[p][i] for p in range(cl.workers)]) for i in range(cl.spec.depth)]
    pre = {}
    for p in range(cl.workers):
        for i in sorted(cl.states[p]):
            try:
                out, _ = kfac_layer_step(cl.states[p][i], caps[p][0][i], caps[p][1][i], agg[i], h, t)
            except OracleError as exc:
                raise type(exc)(f"worker {p}, layer {i}: {exc}") from exc
            pre[i] = out
    for i in range(cl.spec.depth):
        cl.momenta[i] *= mu
        cl.momenta[i] += pre[i]
        cl.weights[i] -= lr * cl.momenta[i]
    return float(np.mean(losses)), pre


def build_mpd_cluster(spec: MlpSpec, workers: int, seed: int, assignment=None) -> Cluster:
    """MPD variants keep averaged factors for EVERY layer on every worker (distsim.py:155-156)."""
    cl = build_cluster(spec, workers, seed, assignment)
    cl.states = [{i: LayerState() for i in range(spec.depth)} for _ in range(workers)]
    return cl


def mpd_kfac_step(cl: Cluster, shards, h: Hyper, lr: float, mu: float, t: int, variant: str = "co"):
    """Model-parallel D-KFAC (distsim.py:341-420): raw local factors of every layer,
    averaged over workers (tree mean), running average on every worker; the owner
    refreshes; "co" broadcasts the decomposition and every worker preconditions
    every layer, "mo" preconditions at the owner and broadcasts the result.  Both
    leave identical replicas, so one weight copy is updated here."""
    from .kfac_ref import apply_preconditioner, compute_factors, factor_due, inverse_due, refresh_inverses, \
        update_running_average
    import copy
    if variant not in ("co", "mo"):
        raise OracleArgumentError(f"unknown mpd variant {variant!r}")
    P, L = cl.workers, cl.spec.depth
    losses, caps, locgrads = [], [], []
    for x, y in shards:
        loss, ins, pgs, gs = forward_backward(cl.spec, cl.weights, x, y)
        losses.append(loss)
        caps.append((ins, pgs))
        locgrads.append(gs)
    agg = [tree_mean([locgrads[p][i] for p in range(P)]) for i in range(L)]
    if factor_due(t, h):
        raw = [[compute_factors(caps[p][0][i], caps[p][1][i]) for i in range(L)] for p in range(P)]
        for i in range(L):
            a_avg = tree_mean([raw[p][i][0] for p in range(P)])
            g_avg = tree_mean([raw[p][i][1] for p in range(P)])
            for p in range(P):
                update_running_average(cl.states[p][i], a_avg, g_avg, h.xi, t)
    owner = {i: p for p, part in enumerate(cl.assignment) for i in part}
    if inverse_due(t, h):
        for i in range(L):
            st = cl.states[owner[i]][i]
            refresh_inverses(st, h, t)
            if variant == "co":
                for p in range(P):
                    if p != owner[i]:
                        d = cl.states[p][i]
                        d.a_eig, d.g_eig = copy.deepcopy(st.a_eig), copy.deepcopy(st.g_eig)
                        d.a_damped_inv = None if st.a_damped_inv is None else st.a_damped_inv.copy()
                        d.g_damped_inv = None if st.g_damped_inv is None else st.g_damped_inv.copy()
                        d.last_inverse_update = t
    if variant == "co":
        pre = {i: apply_preconditioner(cl.states[0][i], agg[i], h) for i in range(L)}
    else:
        pre = {i: apply_preconditioner(cl.states[owner[i]][i], agg[i], h) for i in range(L)}
    for i in range(L):
        cl.momenta[i] *= mu
        cl.momenta[i] += pre[i]
        cl.weights[i] -= lr * cl.momenta[i]
    return float(np.mean(losses)), pre
