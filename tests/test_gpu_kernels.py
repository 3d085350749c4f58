"""GPU parity of every libdpkfac kernel against the float64 oracle (tolerances written per test).

Bar (BASELINE north_star): relative Frobenius error <= 1e-3 for factors and
preconditioned gradients in the fp32/TF32 path."""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import kfac_ref as K

pytestmark = pytest.mark.gpu

TOL = 1e-3


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def dev():
    return torch.device("cuda", 0)


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x)).float().to(dev())


def N(t):
    return t.double().cpu().numpy()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2206_15143_b200 import _lib
    _lib.load()


# ---------------------------------------------------------------- K1 SYRK + EMA
@pytest.mark.parametrize("d,m", [(1, 5), (10, 64), (127, 33), (128, 128), (129, 4000), (300, 777), (785, 64),
                                 (64, 100352)])
@pytest.mark.parametrize("precision", ["tf32", "3xtf32"])
def test_syrk_rows_k_matches_oracle(d, m, precision):
    from paper_2206_15143_b200 import kfac as FK
    rng = np.random.default_rng(d * 7 + m)
    x = rng.standard_normal((d, m))
    g = rng.standard_normal((3, m))
    a, _ = FK.compute_factors(T(x), T(g), precision=precision)
    a_ref, _ = K.compute_factors(x, g)
    # 3xTF32 products are fp32-grade; the bound is fp32 accumulation over up to 1e5 samples
    assert rel(N(a), a_ref) <= (TOL if precision == "tf32" else 5e-5)
    assert torch.equal(a, a.T)  # exactly symmetric like (F + F^T)/2


def test_syrk_ema_fused_running_average():
    from paper_2206_15143_b200 import kfac as FK
    rng = np.random.default_rng(1)
    st_ref, st = K.LayerState(), FK.FactorState()
    for t in range(4):
        x = np.maximum(rng.standard_normal((200, 300)), 0)
        g = rng.standard_normal((50, 300)) * 0.1
        a_new, g_new = K.compute_factors(x, g)
        K.update_running_average(st_ref, a_new, g_new, 0.3, t)
        FK.update_factors_fused(st, T(x), T(g), 0.3, t, precision="3xtf32")
        assert rel(N(st.a_cov), st_ref.a_cov) <= 1e-5
        assert rel(N(st.g_cov), st_ref.g_cov) <= 1e-5
        assert st.last_factor_update == t


def _linear_capture(rng, b, d, bias):
    x = rng.standard_normal((b, d))
    X = x.T
    if bias:
        X = np.vstack([X, np.ones((1, b))])
    return x, X


@pytest.mark.parametrize("b,d,bias", [(64, 784, True), (32, 2048, True), (7, 5, False)])
def test_syrk_rows_mn_linear_input_with_bias_row(b, d, bias):
    from paper_2206_15143_b200 import _lib as L, ops
    rng = np.random.default_rng(b + d)
    x, X = _linear_capture(rng, b, d, bias)
    xt = T(x)
    dd = d + int(bias)
    out = torch.full((dd, dd), float("nan"), device=dev())
    ops.syrk_ema([ops.factor_job(ops.operand_rows_mn(xt, bias), out, 1.0 / b, 0.0)], "tf32")
    torch.cuda.synchronize()
    want, _ = K.compute_factors(X, X[:1])
    assert rel(N(out), want) <= TOL
    assert torch.isfinite(out).all()


@pytest.mark.parametrize("shape,k,s,p,dil", [
    ((2, 3, 9, 9), 3, 1, 1, 1), ((2, 4, 10, 10), 3, 2, 1, 1), ((3, 5, 8, 8), 1, 2, 0, 1),
    ((1, 3, 15, 15), 7, 2, 3, 1), ((2, 2, 9, 9), 3, 1, 2, 2), ((4, 64, 14, 14), 3, 1, 1, 1)])
@pytest.mark.parametrize("channels_last", [False, True])
def test_syrk_implicit_im2col_matches_unfold(shape, k, s, p, dil, channels_last):
    from paper_2206_15143_b200 import ops
    rng = np.random.default_rng(sum(shape) + k)
    x = np.maximum(rng.standard_normal(shape), 0)
    xt = T(x)
    if channels_last:
        xt = xt.to(memory_format=torch.channels_last)
    cols = K.unfold_columns(x, k, k, s, p, dil, bias=True)
    d = cols.shape[0]
    out = torch.empty(d, d, device=dev())
    op = ops.operand_im2col(xt, (k, k), (s, s), (p, p), (dil, dil), bias_row=True)
    assert op.cols == cols.shape[1]
    ops.syrk_ema([ops.factor_job(op, out, 1.0 / cols.shape[1], 0.0)], "3xtf32")
    torch.cuda.synchronize()
    want, _ = K.compute_factors(cols, cols[:1])
    assert rel(N(out), want) <= 1e-5


def test_grouped_syrk_many_problems_and_split_k():
    from paper_2206_15143_b200 import ops
    rng = np.random.default_rng(5)
    jobs, outs, refs, keep = [], [], [], []
    for i in range(45):  # > MAXP per launch -> several launches
        d = int(rng.integers(1, 300))
        m = int(rng.integers(1, 20000)) if i % 5 else 60000
        x = rng.standard_normal((d, m)).astype(np.float32)
        xt = T(x)
        o = torch.empty(d, d, device=dev())
        jobs.append(ops.factor_job(ops.operand_rows_k(xt), o, 1.0 / m, 0.0))
        outs.append(o)
        keep.append(xt)
        refs.append(x.astype(np.float64) @ x.T.astype(np.float64) / m)
    ops.syrk_ema(jobs, "tf32")
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert rel(N(o), r) <= TOL


# ---------------------------------------------------------------- generic GEMM engine
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (130, 70, 45), (512, 785, 300), (1000, 2049, 33)])
def test_gemm_all_operand_majors(m, n, k):
    from paper_2206_15143_b200 import _lib as L, ops
    rng = np.random.default_rng(m + n + k)
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((n, k))
    c = rng.standard_normal((m, n))
    at, bt, ct = T(a), T(b), T(c)
    atr, btr = T(a.T), T(b.T)
    for a_op, b_op in [(ops.operand_rows_k(at), ops.operand_rows_k(bt)),
                       (ops.operand_rows_mn(atr), ops.operand_rows_k(bt)),
                       (ops.operand_rows_k(at), ops.operand_rows_mn(btr)),
                       (ops.operand_rows_mn(atr), ops.operand_rows_mn(btr))]:
        out = torch.empty(m, n, device=dev())
        j = L.GemmJob()
        j.a, j.b = a_op, b_op
        j.out, j.ldo = out.data_ptr(), n
        j.cin, j.ldc = ct.data_ptr(), n
        j.alpha, j.beta = 0.5, -2.0
        ops.gemm([j], "3xtf32")
        torch.cuda.synchronize()
        assert rel(N(out), 0.5 * a @ b.T - 2.0 * c) <= 1e-5


@pytest.mark.parametrize("m,n,k,sym", [(128, 128, 128, False), (64, 200, 300, False), (33, 17, 1, False),
                                       (256, 256, 96, False), (300, 300, 257, True), (128, 128, 33, True)])
def test_gemm_latency_path_exact_fp32(m, n, k, sym):
    """Small 3xtf32 groups run on the CUDA-core latency path (gemm_simt.cu: cp.async
    ring, K from one chunk to past the ring's depth, symmetric lower tiles + mirror):
    exact fp32 products, so within fp32 accumulation error of the float64 product."""
    from paper_2206_15143_b200 import _lib as L, ops
    rng = np.random.default_rng(m * 7 + n + k)
    a = rng.standard_normal((m, k)).astype(np.float32).astype(np.float64)
    b = a if sym else rng.standard_normal((n, k)).astype(np.float32).astype(np.float64)
    c = rng.standard_normal((m, n)).astype(np.float32).astype(np.float64)
    at, bt, ct = T(a), T(b), T(c)
    atr, btr = T(a.T), T(b.T)
    pairs = [(ops.operand_rows_k(at), ops.operand_rows_k(bt)), (ops.operand_rows_mn(atr), ops.operand_rows_mn(btr))]
    for a_op, b_op in pairs:
        out = torch.full((m, n), float("nan"), device=dev())
        j = L.GemmJob()
        j.a, j.b = a_op, b_op
        j.out, j.ldo = out.data_ptr(), n
        j.cin, j.ldc = (0, 0) if sym else (ct.data_ptr(), n)
        j.alpha, j.beta = (0.25, 0.0) if sym else (0.5, -2.0)
        j.symmetric = int(sym)
        ops.gemm([j], "3xtf32")
        torch.cuda.synchronize()
        want = 0.25 * a @ a.T if sym else 0.5 * a @ b.T - 2.0 * c
        assert rel(N(out), want) <= 2e-6, rel(N(out), want)


@pytest.mark.parametrize("scale", [1.0, 3e4, 1e-6])
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (130, 70, 45), (512, 785, 300), (1000, 2049, 33), (600, 600, 700)])
def test_gemm_3xf16_all_operand_majors(m, n, k, scale):
    """DPK_PREC_3XF16: fp16 hi / lo parts of the amax-prescaled operands on kind::f16
    MMAs -- fp32-grade like 3xTF32 for operands far above the fp16 range (3e4 squared
    and beyond 65504 after the product) and far below it (1e-6), single CTAs and
    CTA pairs, every operand major (MN-major tiles go through the plain TMA map)."""
    from paper_2206_15143_b200 import _lib as L, ops
    rng = np.random.default_rng(m + n + k + 1)
    a = rng.standard_normal((m, k)) * scale
    a[:, :1] *= 1e-3  # graded columns: small entries keep their relative accuracy
    b = rng.standard_normal((n, k)) * scale
    c = rng.standard_normal((m, n)) * scale * scale
    at, bt, ct = T(a), T(b), T(c)
    atr, btr = T(a.T), T(b.T)
    for a_op, b_op in [(ops.operand_rows_k(at), ops.operand_rows_k(bt)),
                       (ops.operand_rows_mn(atr), ops.operand_rows_k(bt)),
                       (ops.operand_rows_k(at), ops.operand_rows_mn(btr)),
                       (ops.operand_rows_mn(atr), ops.operand_rows_mn(btr))]:
        out = torch.full((m, n), float("nan"), device=dev())
        j = L.GemmJob()
        j.a, j.b = a_op, b_op
        j.out, j.ldo = out.data_ptr(), n
        j.cin, j.ldc = ct.data_ptr(), n
        j.alpha, j.beta = 0.5, -2.0
        ops.gemm([j], "3xf16")
        torch.cuda.synchronize()
        want = 0.5 * a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T - 2.0 * c
        assert rel(N(out), want) <= 1e-5, rel(N(out), want)


# ---------------------------------------------------------------- K3 damped inverse
def _spd(rng, n, cond_floor=1e-2):
    b = rng.standard_normal((n, n + 3))
    return b @ b.T / (n + 3) + cond_floor * np.eye(n)


@pytest.mark.parametrize("n", [1, 2, 17, 64, 128, 129, 200, 513, 1000, 2049])
def test_spd_inverse_matches_oracle(n):
    from paper_2206_15143_b200 import kfac as FK
    rng = np.random.default_rng(n)
    a = _spd(rng, n)
    got = FK.sym_inverse(T(a))
    want = K.spd_inverse(a)
    cond = np.linalg.cond(a)
    # fp32-grade (3xTF32) elimination: error ~ cond * 2^-23 up to a modest growth factor
    assert rel(N(got), want) <= max(1e-5, 20 * cond * 2.0 ** -23), (rel(N(got), want), cond)
    assert torch.equal(got, got.T)


@pytest.mark.parametrize("d,m,shift", [(1500, 500, 0.045), (4608, 1568, 0.045), (700, 64, 0.01)])
def test_spd_inverse_rank_deficient_factor_plus_damping(d, m, shift):
    """The hard case of real K-FAC factors: X X^T / M has rank M < d, only the damping
    keeps it definite (ResNet-50 layer4 3x3: d=4608, M=1568)."""
    from paper_2206_15143_b200 import kfac as FK
    rng = np.random.default_rng(d)
    x = np.maximum(rng.standard_normal((d, m)), 0).astype(np.float32)
    a = x.astype(np.float64) @ x.T.astype(np.float64) / m + shift * np.eye(d)
    got = FK.sym_inverse(T(a))
    want = np.linalg.inv(a)
    cond = np.linalg.cond(a)
    assert rel(N(got), want) <= max(1e-4, 20 * cond * 2.0 ** -23), (rel(N(got), want), cond)


@pytest.mark.parametrize("n,shift", [(1, 0.5), (37, 0.0), (128, 0.01), (129, 0.02), (513, 0.01), (2049, 0.045),
                                     (4608, 0.045)])
def test_factored_spd_inverse_matches_oracle(n, shift):
    """dpk_chol_factor_inv_batched: X = L^-1 of (A + shift I), lower triangular; X^T X
    is the reference's damped inverse (numerics.sym_inverse of the damped factor)."""
    from paper_2206_15143_b200 import _lib as L, ops
    rng = np.random.default_rng(n + 7)
    m = max(n // 3, 4)
    x = np.maximum(rng.standard_normal((n, m)), 0)
    a = x @ x.T / m + (0.05 if shift == 0.0 else 0.0) * np.eye(n)
    src = T(a)
    dst = torch.full((n, ops.factor_ld(n)), float("nan"), device=dev())[:, :n]
    sh = torch.tensor([shift], device=dev())
    info = torch.zeros(1, dtype=torch.int32, device=dev())
    ops.chol_factor_inv([ops.spd_factor_job(src, dst, sh, info, L.INFO_NOT_SPD_A)])
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    X = N(dst)
    assert np.all(X[np.triu_indices(n, 1)] == 0.0)  # exactly lower triangular
    want = K.spd_inverse(a + shift * np.eye(n))
    cond = np.linalg.cond(a + shift * np.eye(n))
    assert rel(X.T @ X, want) <= max(1e-4, 20 * cond * 2.0 ** -23), (rel(X.T @ X, want), cond)


@pytest.mark.parametrize("precision", ["3xtf32", "3xf16"])
@pytest.mark.parametrize("din,dout,gamma", [(785, 512, 0.03), (65, 9, 0.002), (2049, 1000, 0.002), (3, 2, 0.03),
                                            (4608, 512, 0.002)])
def test_precondition_factored_matches_oracle(din, dout, gamma, precision):
    """dpk_precond_factored with the factors of dpk_chol_factor_inv_batched equals the
    reference's G_inv @ grad @ A_inv (kfac.precondition_inverse, kfac.py:165-171), in
    both fp32-grade precisions (3xF16: amax-prescaled fp16 hi / lo parts)."""
    from paper_2206_15143_b200 import _lib as L, ops
    rng = np.random.default_rng(din * 3 + dout)
    x = np.maximum(rng.standard_normal((din, 256)), 0)
    g = rng.standard_normal((dout, 256)) * 0.1
    grad = rng.standard_normal((dout, din)) * 0.01
    a, gg = K.compute_factors(x, g)
    pi = K.pi_scalar(a, gg)
    sa, sg = pi * np.sqrt(gamma), np.sqrt(gamma) / pi
    xa = torch.zeros(din, ops.factor_ld(din), device=dev())[:, :din]
    xg = torch.zeros(dout, ops.factor_ld(dout), device=dev())[:, :dout]
    shifts = torch.tensor([sa, sg], device=dev(), dtype=torch.float32)
    info = torch.zeros(1, dtype=torch.int32, device=dev())
    ta, tg = T(a), T(gg)  # keep the sources alive: the jobs hold raw pointers
    ops.chol_factor_inv([ops.spd_factor_job(ta, xa, shifts[0], info, L.INFO_NOT_SPD_A),
                         ops.spd_factor_job(tg, xg, shifts[1], info, L.INFO_NOT_SPD_G)])
    gr, out, tmp = T(grad), torch.empty(dout, din, device=dev()), torch.empty(dout, din, device=dev())
    ops.precondition_factored([ops.precond_factor_job(gr, xa, xg, out, tmp)], precision)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    want = K.precondition_inverse(a, gg, grad, gamma)
    assert rel(N(out), want) <= TOL, rel(N(out), want)


def test_damped_inverses_and_pi_match_oracle():
    from paper_2206_15143_b200 import kfac as FK
    rng = np.random.default_rng(3)
    for da, dg, gamma in [(785, 512, 0.03), (147, 64, 0.002), (300, 10, 1.0)]:
        x = np.maximum(rng.standard_normal((da, 600)), 0)
        g = rng.standard_normal((dg, 600)) * 0.01
        a, gg = K.compute_factors(x, g)
        ai, gi = FK.damped_inverses(T(a), T(gg), gamma)
        ai_r, gi_r = K.damped_inverses(a, gg, gamma)
        assert rel(N(ai), ai_r) <= 1e-4 and rel(N(gi), gi_r) <= 1e-4
        assert abs(FK.pi_scalar(T(a), T(gg)) - K.pi_scalar(a, gg)) <= 1e-5 * K.pi_scalar(a, gg)


def test_non_spd_raises_numeric_error_like_reference():
    from paper_2206_15143_b200 import NumericError
    from paper_2206_15143_b200 import kfac as FK
    a = np.eye(150)
    a[70, 70] = -1.0
    with pytest.raises(NumericError, match="not positive definite"):
        FK.sym_inverse(T(a))
    with pytest.raises(NumericError, match="traces must be positive"):
        FK.damped_inverses(T(np.zeros((3, 3))), T(np.eye(2)), 0.03)
    with pytest.raises(NumericError, match="damped input factor A is not invertible"):
        FK.damped_inverses(T(np.diag([1.0, -5.0, 1.0, 1.0])), T(np.eye(2)), 0.0)


# ---------------------------------------------------------------- K4 eigen
@pytest.mark.parametrize("n", [1, 2, 3, 31, 64, 127, 128])
def test_sym_eig_onchip_jacobi(n):
    from paper_2206_15143_b200 import kfac as FK
    rng = np.random.default_rng(n)
    a = _spd(rng, n, 0.0)
    e = FK.sym_eig(T(a))
    r = K.symmetric_eig(a)
    assert rel(N(e.values), r.values) <= 1e-5
    assert np.all(np.diff(N(e.values)) <= 0)
    q = N(e.q)
    assert np.abs(q.T @ q - np.eye(n)).max() <= 1e-4
    assert rel(q @ np.diag(N(e.values)) @ q.T, a) <= 5e-5  # fp32 Jacobi, n <= 128


@pytest.mark.parametrize("n,m", [(129, 400), (200, 60), (256, 1000), (577, 300), (1000, 1568)])
def test_sym_eig_block_jacobi_native(n, m):
    """n > 128: the tensor-core block Jacobi (csrc/syevj.cu) -- no library
    eigensolver.  Rank-deficient K-FAC-like factors (m < n: a cluster of zero
    eigenvalues), odd n (zero padding to a multiple of 128)."""
    from paper_2206_15143_b200 import kfac as FK
    rng = np.random.default_rng(n + m)
    x = np.maximum(rng.standard_normal((n, m)), 0) * np.exp(-np.arange(n) / (n / 3))[:, None]
    a = x @ x.T / m
    e = FK.sym_eig(T(a), solver="native")
    r = K.symmetric_eig(a)
    v, q = N(e.values), N(e.q)
    assert np.all(np.diff(v) <= 0)
    assert np.abs(v - r.values).max() <= 3e-5 * np.abs(r.values).max()
    assert np.abs(q.T @ q - np.eye(n)).max() <= 3e-4
    assert rel(q @ np.diag(v) @ q.T, a) <= 2e-4


@pytest.mark.parametrize("din,dout,gamma", [(577, 256, 0.002), (1153, 512, 0.03)])
def test_precondition_eigen_large_native_matches_oracle(din, dout, gamma):
    from paper_2206_15143_b200 import kfac as FK
    rng = np.random.default_rng(din + 3 * dout)
    x = np.maximum(rng.standard_normal((din, 800)), 0)
    x[-1] = 1.0
    g = rng.standard_normal((dout, 800)) * 0.1
    grad = rng.standard_normal((dout, din)) * 0.01
    a, gg = K.compute_factors(x, g)
    for solver in ("native", "cusolver"):
        got = FK.precondition_eigen(FK.sym_eig(T(a), solver), FK.sym_eig(T(gg), solver), T(grad), gamma)
        want = K.precondition_eigen(K.symmetric_eig(a), K.symmetric_eig(gg), grad, gamma)
        assert rel(N(got), want) <= TOL, (solver, rel(N(got), want))


# ---------------------------------------------------------------- K5 / K6
@pytest.mark.parametrize("din,dout,gamma", [(785, 512, 0.03), (65, 9, 0.002), (2049, 1000, 0.002), (3, 2, 0.03)])
def test_precondition_inverse_matches_oracle(din, dout, gamma):
    from paper_2206_15143_b200 import kfac as FK
    rng = np.random.default_rng(din)
    x = np.maximum(rng.standard_normal((din, 256)), 0)
    g = rng.standard_normal((dout, 256)) * 0.1
    grad = rng.standard_normal((dout, din)) * 0.01
    a, gg = K.compute_factors(x, g)
    got = FK.precondition_inverse(T(a), T(gg), T(grad), gamma)
    want = K.precondition_inverse(a, gg, grad, gamma)
    assert rel(N(got), want) <= TOL


@pytest.mark.parametrize("din,dout,gamma", [(65, 9, 0.002), (128, 100, 0.03), (3, 2, 0.03), (120, 1, 0.5)])
def test_precondition_eigen_matches_oracle(din, dout, gamma):
    from paper_2206_15143_b200 import kfac as FK
    rng = np.random.default_rng(din + dout)
    x = np.maximum(rng.standard_normal((din, 200)), 0)
    g = rng.standard_normal((dout, 200)) * 0.1
    grad = rng.standard_normal((dout, din)) * 0.01
    a, gg = K.compute_factors(x, g)
    got = FK.precondition_eigen(FK.sym_eig(T(a)), FK.sym_eig(T(gg)), T(grad), gamma)
    want = K.precondition_eigen(K.symmetric_eig(a), K.symmetric_eig(gg), grad, gamma)
    assert rel(N(got), want) <= TOL


def test_eigen_zero_denominator_raises():
    from paper_2206_15143_b200 import NumericError
    from paper_2206_15143_b200 import kfac as FK
    z = FK.sym_eig(T(np.zeros((2, 2))))
    with pytest.raises(NumericError, match="denominator"):
        FK.precondition_eigen(z, z, T(np.ones((2, 2))), 0.0)


# ---------------------------------------------------------------- K7 pack / unpack
def test_pack_unpack_roundtrip_with_bias_column():
    from paper_2206_15143_b200 import ops
    rng = np.random.default_rng(9)
    w1 = T(rng.standard_normal((5, 3, 3, 3)))
    w2 = T(rng.standard_normal((4, 7)))
    b2 = T(rng.standard_normal(4))
    w1_0, w2_0, b2_0 = w1.clone(), w2.clone(), b2.clone()
    flat = torch.zeros(5 * 27 + 4 * 8 + 10, device=dev())
    segs = [ops.segment(w1, None, 0), ops.segment(w2, b2, 5 * 27 + 3)]
    ops.pack(segs, flat, 0.5)
    torch.cuda.synchronize()
    assert torch.equal(flat[:135].view(5, 27), 0.5 * w1_0.view(5, 27))
    m2 = flat[138:138 + 32].view(4, 8)
    assert torch.equal(m2[:, :7], 0.5 * w2_0) and torch.equal(m2[:, 7], 0.5 * b2_0)
    flat.mul_(4.0)
    ops.unpack(segs, flat, 1.0)
    torch.cuda.synchronize()
    assert torch.equal(w1, 2.0 * w1_0) and torch.equal(w2, 2.0 * w2_0) and torch.equal(b2, 2.0 * b2_0)


# ---------------------------------------------------------------- tap-major (channels-last) im2col: tiled-TMA tap boxes
# (TMA_TAPS) for NHWC inputs with C % 32 == 0, the producer gather otherwise
def _tap_perm(c, kh, kw):
    """held (kh, kw, c) position t -> reference (c, kh, kw) row index."""
    import numpy as _np
    return _np.arange(c * kh * kw).reshape(c, kh, kw).transpose(1, 2, 0).reshape(-1)


@pytest.mark.parametrize("shape,k,s,p", [((4, 64, 14, 14), 3, 1, 1), ((2, 128, 9, 9), 3, 2, 1),
                                         ((3, 32, 8, 8), 1, 2, 0), ((2, 64, 7, 7), 3, 1, 1),
                                         ((2, 96, 12, 10), 5, 1, 2), ((1, 32, 6, 6), 1, 1, 0),
                                         # tiled-TMA tap boxes: 32 samples per chunk (wb=1),
                                         # 16 x 2 columns, 4 x 8 columns at stride 2, zero-filled
                                         # sample tail (odd output width), 256 channels (4-group box)
                                         ((32, 64, 8, 8), 3, 1, 1), ((16, 32, 10, 10), 3, 1, 1),
                                         ((4, 32, 16, 16), 3, 2, 1), ((16, 32, 7, 7), 3, 1, 1),
                                         ((32, 256, 4, 4), 1, 2, 0), ((8, 128, 6, 6), 7, 1, 3)])
@pytest.mark.parametrize("channels_last", [True, False])
def test_syrk_tapmajor_im2col_matches_unfold(shape, k, s, p, channels_last):
    from paper_2206_15143_b200 import ops
    rng = np.random.default_rng(sum(shape) + 7 * k)
    x = np.maximum(rng.standard_normal(shape), 0)
    xt = T(x)
    if channels_last:  # NHWC with C % 32 == 0 -> TMA tap boxes; otherwise the gather path
        xt = xt.to(memory_format=torch.channels_last)
    cols = K.unfold_columns(x, k, k, s, p)
    perm = _tap_perm(shape[1], k, k)
    d = cols.shape[0]
    for prec, tol in (("tf32", TOL), ("3xtf32", 3e-5)):  # fp32 accumulation over up to 2048 columns per split
        out = torch.full((d, d), float("nan"), device=dev())
        op = ops.operand_im2col(xt, (k, k), (s, s), (p, p), (1, 1), tap_major=True)
        ops.syrk_ema([ops.factor_job(op, out, 1.0 / cols.shape[1], 0.0)], prec)
        torch.cuda.synchronize()
        want, _ = K.compute_factors(cols[perm], cols[:1])
        assert rel(N(out), want) <= tol, (prec, rel(N(out), want))


def test_pack_unpack_tap_major_perm():
    from paper_2206_15143_b200 import ops
    rng = np.random.default_rng(11)
    w = T(rng.standard_normal((6, 5, 3, 3)))
    w0 = w.clone()
    flat = torch.zeros(6 * 45, device=dev())
    ops.pack([ops.segment(w, None, 0, tap_major=True)], flat, 1.0)
    torch.cuda.synchronize()
    assert torch.equal(flat.view(6, 45), w0.permute(0, 2, 3, 1).reshape(6, 45))
    wcl = w0.clone().to(memory_format=torch.channels_last)
    flat2 = torch.zeros_like(flat)
    ops.pack([ops.segment(wcl, None, 0, tap_major=True)], flat2, 1.0)
    torch.cuda.synchronize()
    assert torch.equal(flat2, flat)
    ops.unpack([ops.segment(w, None, 0, tap_major=True)], flat * 3.0, 1.0)
    torch.cuda.synchronize()
    assert torch.equal(w, 3.0 * w0)


@pytest.mark.parametrize("shape,k,s,p,bias", [((2, 64, 9, 9), 3, 1, 1, False), ((2, 3, 15, 15), 7, 2, 3, True),
                                              ((2, 32, 8, 8), 1, 2, 0, False), ((1, 6, 7, 7), 3, 1, 2, True)])
@pytest.mark.parametrize("channels_last,tap", [(True, True), (False, True), (False, False), (True, False)])
def test_im2col_materialize_matches_unfold(shape, k, s, p, bias, channels_last, tap):
    from paper_2206_15143_b200 import ops
    rng = np.random.default_rng(sum(shape) + k + 3 * bias)
    x = rng.standard_normal(shape)
    xt = T(x)
    if channels_last:
        xt = xt.to(memory_format=torch.channels_last)
    op = ops.operand_im2col(xt, (k, k), (s, s), (p, p), (1, 1), bias_row=bias, tap_major=tap)
    d = op.rows + op.bias_row
    ld = (d + 3) // 4 * 4
    out = torch.full((op.cols, ld), float("nan"), device=dev())
    ops.im2col_materialize([(op, out)])
    torch.cuda.synchronize()
    cols = K.unfold_columns(x, k, k, s, p, bias=bias)
    if tap:
        perm = _tap_perm(shape[1], k, k)
        if bias:
            perm = np.concatenate([perm, [cols.shape[0] - 1]])
        cols = cols[perm]
    assert np.array_equal(N(out[:, :d]).T, cols.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("shape,k,s,p,dil", [((32, 64, 9, 9), 3, 1, 2, 2), ((8, 32, 11, 11), 3, 2, 2, 2)])
def test_syrk_taps_dilated_matches_unfold(shape, k, s, p, dil):
    from paper_2206_15143_b200 import ops
    rng = np.random.default_rng(3 + dil)
    x = rng.standard_normal(shape)
    xt = T(x).to(memory_format=torch.channels_last)
    cols = K.unfold_columns(x, k, k, s, p, dil)
    perm = _tap_perm(shape[1], k, k)
    d = cols.shape[0]
    out = torch.full((d, d), float("nan"), device=dev())
    op = ops.operand_im2col(xt, (k, k), (s, s), (p, p), (dil, dil), tap_major=True)
    want, _ = K.compute_factors(cols[perm], cols[:1])
    for prec, tol in (("tf32", TOL), ("3xtf32", 5e-5)):  # fp32 accumulation over M = 2592 / 968 columns
        ops.syrk_ema([ops.factor_job(op, out, 1.0 / cols.shape[1], 0.0)], prec)
        torch.cuda.synchronize()
        assert rel(N(out), want) <= tol, (prec, rel(N(out), want))


# ---------------------------------------------------------------- fp16 feature-major patches + kind::f16 SYRK
@pytest.mark.parametrize("shape,k,s,p,bias,channels_last", [((4, 64, 14, 14), 3, 1, 1, False, True),
                                                           ((3, 32, 9, 9), 3, 2, 1, False, True),
                                                           ((2, 3, 20, 20), 7, 2, 3, False, True),
                                                           ((2, 16, 8, 8), 3, 1, 1, True, False),
                                                           ((32, 256, 7, 7), 1, 2, 0, False, True),
                                                           ((2, 96, 12, 10), 5, 1, 2, False, True),
                                                           # row-staged fp16 kernel: stem-like 7x7/2
                                                           # (OW % 8 == 0), NHWC and NCHW, bias row
                                                           ((2, 3, 32, 32), 7, 2, 3, False, True),
                                                           ((2, 3, 32, 32), 7, 2, 3, True, False),
                                                           # tiled kernel with C % 32 != 0: two taps per
                                                           # 32-row group (C = 16, odd tap count -> a
                                                           # half group), C = 24 / 8 / 48 runs
                                                           ((4, 16, 32, 32), 3, 1, 1, False, True),
                                                           ((3, 16, 15, 17), 3, 2, 1, False, True),
                                                           ((2, 24, 9, 9), 3, 1, 1, False, True),
                                                           ((2, 8, 10, 10), 5, 1, 2, False, True),
                                                           ((2, 48, 7, 7), 3, 1, 1, False, True)])
def test_f16_patches_and_syrk_match_unfold(shape, k, s, p, bias, channels_last):
    from paper_2206_15143_b200 import ops
    rng = np.random.default_rng(sum(shape) + k)
    x = np.maximum(rng.standard_normal(shape), 0)
    xt = T(x)
    if channels_last:
        xt = xt.to(memory_format=torch.channels_last)
    tap = channels_last and k > 1
    op = ops.operand_im2col(xt, (k, k), (s, s), (p, p), (1, 1), bias_row=bias, tap_major=tap)
    cols = K.unfold_columns(x, k, k, s, p, 1, bias)
    perm = _tap_perm(shape[1], k, k) if tap else np.arange(shape[1] * k * k)
    if bias:
        perm = np.concatenate([perm, [cols.shape[0] - 1]])
    want_cols = cols[perm]
    d, M = want_cols.shape
    ld = (M + 7) // 8 * 8
    patch = torch.full((d, ld), float("nan"), dtype=torch.float16, device=dev())
    ops.im2col_materialize_f16([(op, patch)])
    torch.cuda.synchronize()
    got = patch[:, :M].float().cpu().numpy()
    assert np.array_equal(got, torch.from_numpy(want_cols).float().half().float().numpy())  # RN half, bit-exact
    out = torch.full((d, d), float("nan"), device=dev())
    ops.syrk_ema([ops.factor_job(ops.operand_rows_k_f16(patch, M), out, 1.0 / M, 0.0)], "tf32")
    torch.cuda.synchronize()
    want, _ = K.compute_factors(want_cols, want_cols[:1])
    assert rel(N(out), want) <= TOL, rel(N(out), want)


@pytest.mark.parametrize("scale", [1e6, 1e-9, 1.0])
@pytest.mark.parametrize("shape,k,s,p,bias,channels_last", [((4, 64, 14, 14), 3, 1, 1, False, True),
                                                           ((2, 3, 32, 32), 7, 2, 3, False, True),
                                                           ((2, 16, 8, 8), 3, 1, 1, True, False)])
def test_f16_patch_prescale_survives_fp16_range(scale, shape, k, s, p, bias, channels_last):
    """Exact power-of-two prescale from a fused amax (dpk_im2col_amax): activations
    far beyond 65504 (scale 1e6) or far below the fp16 normals (1e-9) give the same
    factor as the float64 reference; the patches hold exactly half(x * 2^-e)."""
    from paper_2206_15143_b200 import ops
    rng = np.random.default_rng(sum(shape) + k + 7)
    x = np.maximum(rng.standard_normal(shape), 0) * scale
    xt = T(x)
    if channels_last:
        xt = xt.to(memory_format=torch.channels_last)
    tap = channels_last and k > 1
    op = ops.operand_im2col(xt, (k, k), (s, s), (p, p), (1, 1), bias_row=bias, tap_major=tap)
    cols = K.unfold_columns(x, k, k, s, p, 1, bias)
    perm = _tap_perm(shape[1], k, k) if tap else np.arange(shape[1] * k * k)
    if bias:
        perm = np.concatenate([perm, [cols.shape[0] - 1]])
    want_cols = cols[perm]
    d, M = want_cols.shape
    ld = (M + 7) // 8 * 8
    patch = torch.full((d, ld), float("nan"), dtype=torch.float16, device=dev())
    amax = torch.full((1,), -1, dtype=torch.int32, device=dev())
    ops.im2col_materialize_f16([(op, patch, amax)])
    torch.cuda.synchronize()
    am = float(np.abs(want_cols.astype(np.float32)).max())
    assert amax.view(torch.float32).item() == am
    e = int(np.floor(np.log2(am))) - 14
    got = patch[:, :M].float().cpu().numpy()
    assert np.isfinite(got).all() and np.abs(got).max() < 2.0 ** 15
    ref = torch.from_numpy(want_cols).float() * (2.0 ** -e)
    assert np.array_equal(got, ref.half().float().numpy())
    out = torch.full((d, d), float("nan"), device=dev())
    for prev in (None, out):  # plain and EMA (beta) epilogues both undo the scale
        a0 = None if prev is None else N(out).copy()
        ops.syrk_ema([ops.factor_job(ops.operand_rows_k_f16(patch, M), out, 1.0 / M, 0.0 if prev is None else 0.5,
                                     x_amax=amax)], "tf32")
        torch.cuda.synchronize()
        want, _ = K.compute_factors(want_cols, want_cols[:1])
        if a0 is not None:
            want = want + 0.5 * a0
        assert rel(N(out), want) <= TOL, rel(N(out), want)


# ---------------------------------------------------------------- non-square kernels / asymmetric padding
# Inception-v4 (config C5): 1x7 / 7x1 convs padded (0,3) / (3,0), 1x3 / 3x1 padded (0,1) / (1,0),
# plus an asymmetric stride -- every im2col form against F.unfold-order columns.
ASYM = [((2, 64, 17, 17), (1, 7), (1, 1), (0, 3)), ((2, 64, 17, 17), (7, 1), (1, 1), (3, 0)),
        ((2, 32, 8, 8), (1, 3), (1, 1), (0, 1)), ((2, 32, 8, 8), (3, 1), (1, 1), (1, 0)),
        ((2, 32, 12, 9), (3, 5), (2, 1), (1, 2)), ((1, 3, 16, 24), (7, 1), (1, 2), (3, 0))]


@pytest.mark.parametrize("shape,kk,ss,pp", ASYM)
@pytest.mark.parametrize("channels_last", [True, False])
def test_asymmetric_kernels_all_im2col_forms_match_unfold(shape, kk, ss, pp, channels_last):
    from paper_2206_15143_b200 import ops
    rng = np.random.default_rng(sum(shape) + 3 * kk[0] + kk[1])
    x = np.maximum(rng.standard_normal(shape), 0)
    xt = T(x)
    if channels_last:
        xt = xt.to(memory_format=torch.channels_last)
    cols = K.unfold_columns(x, kk[0], kk[1], ss, pp)
    d, M = cols.shape
    for tap in (False, True):
        perm = _tap_perm(shape[1], kk[0], kk[1]) if tap else np.arange(d)
        want_cols = cols[perm]
        want, _ = K.compute_factors(want_cols, want_cols[:1])
        op = ops.operand_im2col(xt, kk, ss, pp, (1, 1), tap_major=tap)
        assert op.cols == M
        # implicit im2col SYRK (gather / TMA tap boxes)
        out = torch.full((d, d), float("nan"), device=dev())
        ops.syrk_ema([ops.factor_job(op, out, 1.0 / M, 0.0)], "3xtf32")
        torch.cuda.synchronize()
        assert rel(N(out), want) <= 1e-5, ("implicit", tap, rel(N(out), want))
        # fp32 sample-major patches, bit-exact
        ld = (d + 3) // 4 * 4
        pm = torch.full((M, ld), float("nan"), device=dev())
        ops.im2col_materialize([(op, pm)])
        torch.cuda.synchronize()
        assert np.array_equal(N(pm[:, :d]).T, want_cols.astype(np.float32).astype(np.float64)), ("f32", tap)
        # fp16 feature-major patches (prescaled), kind::f16 SYRK
        p16 = torch.full((d, (M + 7) // 8 * 8), float("nan"), dtype=torch.float16, device=dev())
        amax = torch.zeros(1, dtype=torch.int32, device=dev())
        ops.im2col_materialize_f16([(op, p16, amax)])
        out.fill_(float("nan"))
        ops.syrk_ema([ops.factor_job(ops.operand_rows_k_f16(p16, M), out, 1.0 / M, 0.0, x_amax=amax)], "tf32")
        torch.cuda.synchronize()
        assert rel(N(out), want) <= TOL, ("f16", tap, rel(N(out), want))


@pytest.mark.parametrize("shape,k,s,p,bias,channels_last", [((2, 8, 12, 12), 3, 1, 1, True, False),
                                                           ((2, 64, 9, 9), (1, 7), 1, (0, 3), False, True),
                                                           ((3, 16, 10, 10), 5, 2, 2, False, False)])
def test_compute_conv_input_factor_matches_unfold(shape, k, s, p, bias, channels_last):
    """kfac.compute_conv_input_factor: the K2 entry point (dpk_conv_im2col_syrk_ema) on a
    conv input, reference (C, kh, kw) row order, against compute_factors on F.unfold
    columns."""
    from paper_2206_15143_b200 import kfac as FK
    rng = np.random.default_rng(sum(shape))
    x = np.maximum(rng.standard_normal(shape), 0)
    xt = T(x)
    if channels_last:
        xt = xt.to(memory_format=torch.channels_last)
    kk = k if isinstance(k, tuple) else (k, k)
    a = FK.compute_conv_input_factor(xt, kk, s, p, bias=bias)
    torch.cuda.synchronize()
    cols = K.unfold_columns(x, kk[0], kk[1], s, p, 1, bias)
    want, _ = K.compute_factors(cols, cols[:1])
    assert rel(N(a), want) <= 1e-5, rel(N(a), want)


@pytest.mark.parametrize("scale", [1.0, 1e6])
@pytest.mark.parametrize("shape,k,s,p", [((4, 64, 14, 14), 3, 1, 1), ((3, 128, 9, 11), 3, 2, 1),
                                         ((2, 64, 12, 12), 1, 2, 0), ((5, 192, 7, 7), 3, 1, 1),
                                         ((2, 64, 17, 17), (1, 7), 1, (0, 3)), ((2, 256, 6, 6), 3, 1, 1)])
def test_implicit_f16_syrk_matches_unfold(shape, k, s, p, scale):
    """DPK_OPND_IM2COL_TAPMAJOR_F16: the channels-last input copied once as prescaled
    fp16 (dpk_im2col_convert_f16, bit-exact half(x * 2^-e)), the patches gathered by
    TMA im2col boxes (64 pixels x 64 channels) inside the kind::f16 SYRK -- equal to
    the fp16-patch route's factor and within TOL of the float64 reference; pixel
    tails (M % 64 != 0), strides, 1x7 kernels and C = 192 / 256 (several 64-row
    groups per tap) included."""
    from paper_2206_15143_b200 import ops
    kh, kw = (k, k) if isinstance(k, int) else k
    ph, pw = (p, p) if isinstance(p, int) else p
    rng = np.random.default_rng(sum(shape) + kh * kw)
    x = np.maximum(rng.standard_normal(shape), 0) * scale
    xt = T(x).to(memory_format=torch.channels_last)
    op = ops.operand_im2col(xt, (kh, kw), (s, s), (ph, pw), (1, 1), tap_major=True)
    n, c, h, w = shape
    x16 = torch.full((n, h, w, c), float("nan"), dtype=torch.float16, device=dev())
    amax = torch.zeros(1, dtype=torch.int32, device=dev())
    ops.im2col_materialize_f16([(op, x16, amax)])
    torch.cuda.synchronize()
    e = int(np.floor(np.log2(np.abs(x.astype(np.float32)).max()))) - 14
    want16 = torch.from_numpy(x.astype(np.float32) * 2.0 ** -e).half().permute(0, 2, 3, 1)
    assert torch.equal(x16.cpu(), want16)  # RN half of the exactly prescaled input
    cols = K.unfold_columns(x, kh, kw, s, p if isinstance(p, int) else (ph, pw))
    perm = _tap_perm(c, kh, kw)
    M = cols.shape[1]
    out = torch.full((op.rows, op.rows), float("nan"), device=dev())
    ops.syrk_ema([ops.factor_job(ops.operand_im2col_f16(op, x16), out, 1.0 / M, 0.0, x_amax=amax)], "tf32")
    # the materialized fp16 route on the same values
    ld = (M + 7) // 8 * 8
    patch = torch.empty(op.rows, ld, dtype=torch.float16, device=dev())
    amax2 = torch.zeros(1, dtype=torch.int32, device=dev())
    ops.im2col_materialize_f16([(op, patch, amax2)])
    ref16 = torch.full_like(out, float("nan"))
    ops.syrk_ema([ops.factor_job(ops.operand_rows_k_f16(patch, M), ref16, 1.0 / M, 0.0, x_amax=amax2)], "tf32")
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    assert rel(N(out), N(ref16)) <= 1e-6, rel(N(out), N(ref16))
    want, _ = K.compute_factors(cols[perm], cols[:1])
    assert rel(N(out), want) <= TOL, rel(N(out), want)


def test_launch_cap_gives_identical_results():
    """dpk_set_launch_cap (ops.launch_cap): fewer persistent CTAs walk the same units --
    the result is bit-identical, and the cap is thread-local and reset on exit."""
    from paper_2206_15143_b200 import _lib as L, ops
    rng = np.random.default_rng(5)
    a, b = T(rng.standard_normal((1000, 700))), T(rng.standard_normal((900, 700)))
    outs = []
    for cap in (0, 16, 3):
        out = torch.empty(1000, 900, device=dev())
        j = L.GemmJob()
        j.a, j.b = ops.operand_rows_k(a), ops.operand_rows_k(b)
        j.out, j.ldo, j.alpha = out.data_ptr(), 900, 1.0
        with ops.launch_cap(cap):
            ops.gemm([j], "3xtf32")
        outs.append(out)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    assert ops.lib().dpk_set_launch_cap(-1) != 0  # invalid


def test_peer_gather_copies_every_source_in_rank_order():
    """dpk_peer_gather (the NVLink all-gather of DPKFAC(peer_gather=True)) on local
    sources: dst = concat(sources), bit-exact; bad counts are rejected like the C ABI says."""
    import ctypes as C
    from paper_2206_15143_b200 import ops
    from paper_2206_15143_b200.errors import ArgumentError
    for n_src, count in ((1, 4), (3, 1000), (4, 25557032 // 4 // 4 * 4), (8, 64)):
        srcs = [torch.randn(count, device=dev()) for _ in range(n_src)]
        dst = torch.full((n_src * count,), float("nan"), device=dev())
        ptrs = (C.c_void_p * n_src)(*[s.data_ptr() for s in srcs])
        ops.peer_gather(dst, ptrs, n_src, count)
        torch.cuda.synchronize()
        assert torch.equal(dst, torch.cat(srcs))
    ptrs = (C.c_void_p * 1)(srcs[0].data_ptr())
    with pytest.raises(ArgumentError):
        ops.peer_gather(dst, ptrs, 1, 6)
