"""Generate golden vectors from the REFERENCE implementation (kfaclab 0.1.0).

Run in the build container, where the read-only reference lives:

    python tests/golden/make_golden.py

It imports ``kfaclab`` from /root/reference/pkg/src (never copied), runs the
reference's own functions on seeded inputs and writes small fixtures next to
this script.  The GPU box never needs /root/reference: tests only read the
committed ``*.npz`` / ``*.json`` files.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import kfaclab  # noqa: F401
    from kfaclab import costmodel, distsim, kfac, model, numerics
    return costmodel, distsim, kfac, model, numerics


# layer cases: (name, d_in, d_out, M, gamma, relu_inputs)
LAYER_CASES = [
    ("tiny", 3, 2, 5, 0.03, False),
    ("mlp_like", 33, 17, 64, 0.03, True),
    ("wide_g", 20, 48, 40, 0.002, False),
    ("tall_a", 65, 9, 130, 0.002, True),
    ("single_sample", 7, 4, 1, 0.5, False),
    ("g_scalar", 12, 1, 24, 0.03, True),
]


def layer_vectors(kfac, numerics):
    out = {}
    for idx, (name, din, dout, m, gamma, relu) in enumerate(LAYER_CASES):
        rng = np.random.default_rng(1000 + idx)
        x = rng.standard_normal((din, m))
        if relu:
            x = np.maximum(x, 0.0)
            x[-1, :] = 1.0  # homogeneous bias row, last
        gam = rng.standard_normal((dout, m)) * 0.1
        grad = rng.standard_normal((dout, din)) * 0.01
        a, g = kfac.compute_factors(x, gam)
        pi = kfac.pi_scalar(a, g)
        a_inv, g_inv = kfac.damped_inverses(a, g, gamma)
        p_inv = kfac.precondition_inverse(a, g, grad, gamma)
        ea, eg = numerics.sym_eig(a), numerics.sym_eig(g)
        p_eig = kfac.precondition_eigen(ea, eg, grad, gamma)
        for key, val in dict(x=x, gam=gam, grad=grad, a=a, g=g, pi=np.array(pi),
                             gamma=np.array(gamma), a_inv=a_inv, g_inv=g_inv,
                             p_inv=p_inv, a_vals=ea.values, g_vals=eg.values,
                             p_eig=p_eig).items():
            out[f"{name}/{key}"] = val
    return out


# multi-step sequences: (name, d_in, d_out, M, hyper kwargs, steps)
SEQ_CASES = [
    ("eig_f1k1", 10, 6, 16, dict(gamma=0.03, xi=0.95, inv_type="eigen", f_freq=1, k_freq=1), 4),
    ("inv_f1k1", 10, 6, 16, dict(gamma=0.03, xi=0.95, inv_type="inverse", f_freq=1, k_freq=1), 4),
    ("inv_f2k3", 9, 5, 12, dict(gamma=0.01, xi=0.3, inv_type="inverse", f_freq=2, k_freq=3), 7),
    ("eig_f3k2", 9, 5, 12, dict(gamma=0.01, xi=0.05, inv_type="eigen", f_freq=3, k_freq=2), 7),
]


def sequence_vectors(kfac):
    out = {}
    for idx, (name, din, dout, m, hk, steps) in enumerate(SEQ_CASES):
        rng = np.random.default_rng(2000 + idx)
        hyper = kfac.KfacHyper(**hk)
        st = kfac.FactorState()
        for t in range(steps):
            x = rng.standard_normal((din, m))
            gam = rng.standard_normal((dout, m))
            grad = rng.standard_normal((dout, din))
            pg, st = kfac.kfac_layer_step(st, x, gam, grad, hyper, t)
            out[f"{name}/{t}/x"] = x
            out[f"{name}/{t}/gam"] = gam
            out[f"{name}/{t}/grad"] = grad
            out[f"{name}/{t}/out"] = pg
            out[f"{name}/{t}/a_cov"] = st.a_cov
            out[f"{name}/{t}/g_cov"] = st.g_cov
            out[f"{name}/{t}/last"] = np.array([st.last_factor_update, st.last_inverse_update])
        out[f"{name}/hyper"] = np.array(json.dumps(hk))
        out[f"{name}/steps"] = np.array(steps)
    return out


MLP_SPEC = dict(dims=(20, 16, 12, 5), activation="relu", bias=True)
MLP_RUNS = [(1, "inverse"), (2, "inverse"), (4, "eigen"), (2, "eigen")]


def mlp_vectors(distsim, kfac, model):
    spec = model.NetworkSpec(MLP_SPEC["dims"], activation="relu",
                             loss_kind="softmax_cross_entropy", bias_mode="homogeneous")
    out = {}
    rng = np.random.default_rng(77)
    steps = 4
    batches = [(rng.standard_normal((20, 16)), rng.integers(0, 5, size=16)) for _ in range(steps)]
    for bi, (x, y) in enumerate(batches):
        out[f"batch/{bi}/x"] = x
        out[f"batch/{bi}/y"] = y
    for workers, inv in MLP_RUNS:
        hyper = kfac.KfacHyper(gamma=0.05, xi=0.9, inv_type=inv, f_freq=1, k_freq=2)
        cl = distsim.build_cluster(spec, "dp_kfac", workers, seed=5)
        losses = []
        for t, (x, y) in enumerate(batches):
            res = distsim.dp_kfac_step(cl, distsim.shard_batch(model.Batch(x, y), workers),
                                       hyper, 0.1, 0.9, t)
            losses.append(res.loss)
        key = f"run/{workers}/{inv}"
        out[key + "/losses"] = np.array(losses)
        for i, layer in enumerate(cl.workers[0].replica.layers):
            out[key + f"/w{i}"] = layer.weight
    return out


def partition_vectors(costmodel, distsim):
    table = {}
    for L in (1, 3, 5, 7, 32, 54, 201):
        for P in (1, 2, 3, 4, 8, 64):
            table[f"{L}x{P}"] = [list(p) for p in distsim.assign_layers_round_robin(L, P)]
    return table


def manifest_vectors(costmodel):
    layers = costmodel.resnet50_layers() if hasattr(costmodel, "resnet50_layers") else None
    if layers is None:
        layers = costmodel.resolve_manifest("resnet50")
    dims = [[int(l.d_in), int(l.d_out)] for l in layers]
    n_g, n_f = costmodel.totals(layers)
    return {"dims": dims, "n_g": int(n_g), "n_f": int(n_f)}


def main():
    costmodel, distsim, kfac, model, numerics = _ref()
    np.savez_compressed(os.path.join(HERE, "kfac_layer.npz"), **layer_vectors(kfac, numerics))
    np.savez_compressed(os.path.join(HERE, "kfac_sequences.npz"), **sequence_vectors(kfac))
    np.savez_compressed(os.path.join(HERE, "mlp_dpkfac.npz"), **mlp_vectors(distsim, kfac, model))
    with open(os.path.join(HERE, "partitions.json"), "w") as f:
        json.dump(partition_vectors(costmodel, distsim), f, indent=0, sort_keys=True)
    with open(os.path.join(HERE, "resnet50_manifest.json"), "w") as f:
        json.dump(manifest_vectors(costmodel), f, indent=0)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
