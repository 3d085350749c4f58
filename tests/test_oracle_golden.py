"""Pin the CPU oracle (oracle/) to golden vectors produced by the reference itself.

The fixtures come from tests/golden/make_golden.py, which ran kfaclab 0.1.0's
own functions; the oracle must reproduce them to float64 rounding.
"""

import json
import os

import numpy as np
import pytest

from oracle import kfac_ref as K
from oracle import mlp_ref as MLP

from conftest import GOLDEN


def _load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def _close(a, b, tol):
    a, b = np.asarray(a), np.asarray(b)
    scale = max(1.0, float(np.abs(b).max()))
    assert np.abs(a - b).max() <= tol * scale, (np.abs(a - b).max(), scale)


@pytest.mark.parametrize("case", ["tiny", "mlp_like", "wide_g", "tall_a", "single_sample", "g_scalar"])
def test_layer_functions_match_reference(case):
    z = _load("kfac_layer.npz")
    g = lambda k: z[f"{case}/{k}"]
    a, gg = K.compute_factors(g("x"), g("gam"))
    _close(a, g("a"), 1e-14)
    _close(gg, g("g"), 1e-14)
    assert np.array_equal(a, a.T) and np.array_equal(gg, gg.T)
    gamma = float(g("gamma"))
    assert abs(K.pi_scalar(a, gg) - float(g("pi"))) <= 1e-13 * float(g("pi"))
    ai, gi = K.damped_inverses(a, gg, gamma)
    _close(ai, g("a_inv"), 1e-11)
    _close(gi, g("g_inv"), 1e-11)
    _close(K.precondition_inverse(a, gg, g("grad"), gamma), g("p_inv"), 1e-11)
    ea, eg = K.symmetric_eig(a), K.symmetric_eig(gg)
    _close(ea.values, g("a_vals"), 1e-12)
    _close(eg.values, g("g_vals"), 1e-12)
    assert np.all(np.diff(ea.values) <= 0)
    _close(K.precondition_eigen(ea, eg, g("grad"), gamma), g("p_eig"), 1e-10)


@pytest.mark.parametrize("case", ["eig_f1k1", "inv_f1k1", "inv_f2k3", "eig_f3k2"])
def test_layer_step_sequences_match_reference(case):
    z = _load("kfac_sequences.npz")
    hk = json.loads(str(z[f"{case}/hyper"]))
    h = K.Hyper(**hk)
    st = K.LayerState()
    for t in range(int(z[f"{case}/steps"])):
        out, st = K.kfac_layer_step(st, z[f"{case}/{t}/x"], z[f"{case}/{t}/gam"],
                                    z[f"{case}/{t}/grad"], h, t)
        _close(out, z[f"{case}/{t}/out"], 1e-10)
        _close(st.a_cov, z[f"{case}/{t}/a_cov"], 1e-13)
        _close(st.g_cov, z[f"{case}/{t}/g_cov"], 1e-13)
        assert [st.last_factor_update, st.last_inverse_update] == list(z[f"{case}/{t}/last"])


def test_partitions_match_reference_bit_exact():
    with open(os.path.join(GOLDEN, "partitions.json")) as f:
        table = json.load(f)
    for key, parts in table.items():
        L, P = map(int, key.split("x"))
        got = K.round_robin_partition(L, P)
        assert [list(p) for p in got] == parts, key
        K.validate_partition(got, L)


def test_known_answer_partitions():
    # reference test_distsim.py:40-57
    assert K.round_robin_partition(4, 4) == ((0,), (1,), (2,), (3,))
    assert K.round_robin_partition(5, 2) == ((0, 2, 4), (1, 3))
    with pytest.raises(K.OracleArgumentError):
        K.validate_partition(((0, 1), (1,)), 2)
    with pytest.raises(K.OracleArgumentError):
        K.validate_partition(((0,), ()), 2)


def test_resnet50_manifest_totals():
    with open(os.path.join(GOLDEN, "resnet50_manifest.json")) as f:
        m = json.load(f)
    assert len(m["dims"]) == 54
    assert m["n_g"] == 25_503_912 and m["n_f"] == 153_851_562  # reference test_cli.py:134-135
    assert sum(a * b for a, b in m["dims"]) == m["n_g"]


@pytest.mark.parametrize("workers,inv", [(1, "inverse"), (2, "inverse"), (4, "eigen"), (2, "eigen")])
def test_mlp_dp_kfac_matches_reference(workers, inv):
    z = _load("mlp_dpkfac.npz")
    spec = MLP.MlpSpec((20, 16, 12, 5), "relu", "softmax_cross_entropy", True)
    h = K.Hyper(gamma=0.05, xi=0.9, inv_type=inv, f_freq=1, k_freq=2)
    cl = MLP.build_cluster(spec, workers, seed=5)
    losses = []
    for t in range(4):
        x, y = z[f"batch/{t}/x"], z[f"batch/{t}/y"]
        loss, _ = MLP.dp_kfac_step(cl, MLP.shard(x, y, workers), h, 0.1, 0.9, t)
        losses.append(loss)
    key = f"run/{workers}/{inv}"
    _close(np.array(losses), z[key + "/losses"], 1e-12)
    for i in range(3):
        _close(cl.weights[i], z[key + f"/w{i}"], 1e-10)


def test_known_answers():
    # reference test_kfac.py:14-19, 85-93, 107-113, 156-169
    a, g = K.compute_factors(np.eye(2), np.array([[1.0, 1.0]]))
    assert np.allclose(a, 0.5 * np.eye(2)) and np.allclose(g, [[1.0]])
    assert abs(K.pi_scalar(np.diag([2.0] * 4), np.diag([1.0, 1.0])) - np.sqrt(2.0)) <= 1e-15
    av, gv, x, gamma = 2.0, 0.5, 3.0, 0.03
    pi = np.sqrt(av / gv)
    want = x / ((gv + np.sqrt(gamma) / pi) * (av + pi * np.sqrt(gamma)))
    got = K.precondition_inverse(np.array([[av]]), np.array([[gv]]), np.array([[x]]), gamma)
    assert abs(got[0, 0] - want) <= 1e-14
    with pytest.raises(K.OracleNumericError):
        K.pi_scalar(np.zeros((2, 2)), np.eye(2))
    with pytest.raises(K.OracleOrderingError):
        K.refresh_inverses(K.LayerState(), K.Hyper(), 0)


def test_unfold_matches_torch():
    torch = pytest.importorskip("torch")
    import torch.nn.functional as F
    rng = np.random.default_rng(3)
    for (kh, s, p) in [(3, 1, 1), (3, 2, 1), (1, 2, 0), (7, 2, 3)]:
        x = rng.standard_normal((2, 3, 9, 9))
        cols = K.unfold_columns(x, kh, kh, s, p)
        t = F.unfold(torch.from_numpy(x), kh, padding=p, stride=s)  # N, C*k*k, L
        want = t.permute(1, 0, 2).reshape(t.shape[1], -1).numpy()
        assert np.array_equal(cols, want)


@pytest.mark.parametrize("workers,variant,inv", [(2, "co", "inverse"), (2, "mo", "inverse"), (4, "co", "eigen"),
                                                 (2, "mo", "eigen"), (1, "co", "inverse")])
def test_mlp_mpd_kfac_matches_reference(workers, variant, inv):
    z = _load("mlp_mpd.npz")
    spec = MLP.MlpSpec((20, 16, 12, 5), "relu", "softmax_cross_entropy", True)
    h = K.Hyper(gamma=0.05, xi=0.9, inv_type=inv, f_freq=1, k_freq=2)
    cl = MLP.build_mpd_cluster(spec, workers, seed=5)
    losses = []
    for t in range(4):
        x, y = z[f"batch/{t}/x"], z[f"batch/{t}/y"]
        loss, _ = MLP.mpd_kfac_step(cl, MLP.shard(x, y, workers), h, 0.1, 0.9, t, variant)
        losses.append(loss)
    key = f"run/{workers}/{variant}/{inv}"
    _close(np.array(losses), z[key + "/losses"], 1e-12)
    for i in range(3):
        _close(cl.weights[i], z[key + f"/w{i}"], 1e-10)
