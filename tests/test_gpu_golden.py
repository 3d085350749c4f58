"""The GPU path over the REFERENCE's own golden vectors (tests/golden/make_golden.py
ran kfaclab 0.1.0 itself to write them; test_oracle_golden.py pins the oracle to
the same files on the CPU).

* kfac_layer.npz -- six per-layer cases (tiny, mlp_like, wide_g, tall_a,
  single_sample, g_scalar): compute_factors, pi_scalar, damped_inverses,
  precondition_inverse, sym_eig (values), precondition_eigen through the
  functional mirror ``paper_2206_15143_b200.kfac`` (kfac.py:85-191,
  numerics.py:75-114); reference test_kfac.py:14-203 is the model.
* kfac_sequences.npz -- multi-step ``kfac_layer_step`` runs with stale FIMs
  (F=1/K=1, F=2/K=3, F=3/K=2; kfac.py:77-82, 257-276; reference
  test_kfac.py:253-283): the preconditioned output, the running-average factors
  and (last_factor_update, last_inverse_update) after every step.

Bar: relative Frobenius error <= 1e-3 (fp32 path; BASELINE north_star), the
integer counters exact.  Precision is the library default ("auto": 3xTF32
factors in eigen mode, 1-pass TF32 in inverse mode).
"""

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
TOL = 1e-3

LAYER_CASES = ["tiny", "mlp_like", "wide_g", "tall_a", "single_sample", "g_scalar"]
SEQ_CASES = ["eig_f1k1", "inv_f1k1", "inv_f2k3", "eig_f3k2"]


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def layer_npz(golden_dir):
    return np.load(os.path.join(golden_dir, "kfac_layer.npz"))


@pytest.fixture(scope="module")
def seq_npz(golden_dir):
    return np.load(os.path.join(golden_dir, "kfac_sequences.npz"))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).float().cuda()


def host(t):
    return t.double().cpu().numpy()


@pytest.mark.parametrize("case", LAYER_CASES)
@pytest.mark.parametrize("precision", ["tf32", "3xtf32"])
def test_compute_factors_and_pi_match_reference_golden(layer_npz, case, precision):
    from paper_2206_15143_b200 import kfac
    g = lambda k: layer_npz[f"{case}/{k}"]
    a, gg = kfac.compute_factors(dev(g("x")), dev(g("gam")), precision=precision)
    assert rel(host(a), g("a")) <= TOL, rel(host(a), g("a"))
    assert rel(host(gg), g("g")) <= TOL, rel(host(gg), g("g"))
    assert torch.equal(a, a.T) and torch.equal(gg, gg.T)  # explicitly symmetric (kfac.py:102-104)
    pi = kfac.pi_scalar(a, gg)
    assert abs(pi - float(g("pi"))) <= TOL * abs(float(g("pi")))


@pytest.mark.parametrize("case", LAYER_CASES)
def test_damped_inverses_and_precondition_inverse_match_reference_golden(layer_npz, case):
    from paper_2206_15143_b200 import kfac
    g = lambda k: layer_npz[f"{case}/{k}"]
    gamma = float(g("gamma"))
    a, gg = dev(g("a")), dev(g("g"))
    a_inv, g_inv = kfac.damped_inverses(a, gg, gamma)
    assert rel(host(a_inv), g("a_inv")) <= TOL, rel(host(a_inv), g("a_inv"))
    assert rel(host(g_inv), g("g_inv")) <= TOL, rel(host(g_inv), g("g_inv"))
    p = kfac.precondition_inverse(a, gg, dev(g("grad")), gamma)
    assert rel(host(p), g("p_inv")) <= TOL, rel(host(p), g("p_inv"))


@pytest.mark.parametrize("case", LAYER_CASES)
def test_sym_eig_and_precondition_eigen_match_reference_golden(layer_npz, case):
    from paper_2206_15143_b200 import kfac
    g = lambda k: layer_npz[f"{case}/{k}"]
    gamma = float(g("gamma"))
    ea, eg = kfac.sym_eig(dev(g("a"))), kfac.sym_eig(dev(g("g")))
    # descending order, orthonormal columns (numerics.py:75-97)
    for e, want in ((ea, g("a_vals")), (eg, g("g_vals"))):
        v = host(e.values)
        assert np.all(np.diff(v) <= 0)
        assert np.abs(v - want).max() <= TOL * max(np.abs(want).max(), 1e-30)
        q = host(e.q)
        assert np.abs(q.T @ q - np.eye(q.shape[0])).max() <= 1e-5
    p = kfac.precondition_eigen(ea, eg, dev(g("grad")), gamma)
    assert rel(host(p), g("p_eig")) <= TOL, rel(host(p), g("p_eig"))


@pytest.mark.parametrize("case", SEQ_CASES)
def test_kfac_layer_step_sequences_with_stale_fim_match_reference_golden(seq_npz, case):
    """F/K staleness: factors refreshed every F steps, decompositions every K, the
    preconditioner always applied with the newest (possibly stale) state."""
    from paper_2206_15143_b200 import kfac
    hk = json.loads(str(seq_npz[f"{case}/hyper"]))
    hyper = kfac.KfacHyper(**hk)
    st = kfac.FactorState()
    for t in range(int(seq_npz[f"{case}/steps"])):
        g = lambda k: seq_npz[f"{case}/{t}/{k}"]
        out, st = kfac.kfac_layer_step(st, dev(g("x")), dev(g("gam")), dev(g("grad")), hyper, t)
        assert rel(host(out), g("out")) <= TOL, (t, rel(host(out), g("out")))
        assert rel(host(st.a_cov), g("a_cov")) <= TOL, (t, rel(host(st.a_cov), g("a_cov")))
        assert rel(host(st.g_cov), g("g_cov")) <= TOL, (t, rel(host(st.g_cov), g("g_cov")))
        assert [st.last_factor_update, st.last_inverse_update] == [int(v) for v in g("last")], t
        if hyper.inv_type == "eigen":
            assert st.a_eig is not None and st.a_damped_inv is None
        else:
            assert st.a_damped_inv is not None and st.a_eig is None
