"""float64 restatement of the reference K-FAC hot path (TEST INFRASTRUCTURE ONLY).

Each function cites the reference lines whose behaviour it reproduces.  The
arithmetic is the same LAPACK-backed numpy/scipy route the reference takes
(``eigh`` for the eigen route, a lower Cholesky plus triangular solves for the
inverse route), so results agree with the reference to rounding; the golden
tests in ``tests/test_oracle_golden.py`` pin that.

Conventions (reference numerics.py:1-16, model.py:9-17):
  * captures are column-per-sample: X is d_in x M, Gamma is d_out x M;
  * gradients are d_out x d_in, G acts on the left, A on the right;
  * the homogeneous bias row of X is the LAST row.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import scipy.linalg


class OracleError(Exception):
    """Base of the oracle's error classes (mirror of reference errors.py:9)."""


class OracleArgumentError(OracleError, ValueError):
    """reference errors.py:17 (ArgumentError)."""


class OracleShapeError(OracleError, ValueError):
    """reference errors.py:13 (ShapeError)."""


class OracleNumericError(OracleError, ArithmeticError):
    """reference errors.py:25 (NumericError)."""


class OracleOrderingError(OracleError, RuntimeError):
    """reference errors.py:29 (OrderingError)."""


# --------------------------------------------------------------------------
# hyper-parameters and state


@dataclass(frozen=True)
class Hyper:
    """reference kfac.py:55-74 -- defaults 0.03 / 0.95 / eigen / 1 / 1."""

    gamma: float = 0.03
    xi: float = 0.95
    inv_type: str = "eigen"
    f_freq: int = 1
    k_freq: int = 1

    def __post_init__(self):
        if not self.gamma >= 0:
            raise OracleArgumentError("damping gamma must be >= 0")
        if not 0.0 < self.xi <= 1.0:
            raise OracleArgumentError("running-average weight xi must lie in (0, 1]")
        if self.inv_type not in ("inverse", "eigen"):
            raise OracleArgumentError("inv_type must be one of ('inverse', 'eigen')")
        if min(self.f_freq, self.k_freq) < 1:
            raise OracleArgumentError("f_freq and k_freq must be >= 1")


@dataclass
class Eig:
    """Columns of ``q`` are eigenvectors; ``values`` descending (numerics.py:33-37)."""

    q: np.ndarray
    values: np.ndarray


@dataclass
class LayerState:
    """reference kfac.py:39-52 (FactorState)."""

    a_cov: Optional[np.ndarray] = None
    g_cov: Optional[np.ndarray] = None
    a_eig: Optional[Eig] = None
    g_eig: Optional[Eig] = None
    a_damped_inv: Optional[np.ndarray] = None
    g_damped_inv: Optional[np.ndarray] = None
    last_factor_update: int = -1
    last_inverse_update: int = -1
    initialized: bool = False


def factor_due(t: int, h: Hyper) -> bool:
    """reference kfac.py:77-78."""
    return t % h.f_freq == 0


def inverse_due(t: int, h: Hyper) -> bool:
    """reference kfac.py:81-82."""
    return t % h.k_freq == 0


# --------------------------------------------------------------------------
# dense linear algebra (reference numerics.py:75-114)


def symmetric_eig(m: np.ndarray) -> Eig:
    """Symmetrize, ``eigh``, reorder to descending (numerics.py:75-97)."""
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise OracleShapeError("sym_eig: expected a square matrix")
    w, v = np.linalg.eigh(0.5 * (m + m.T))
    w = np.ascontiguousarray(w[::-1])
    v = np.ascontiguousarray(v[:, ::-1])
    if not (np.all(np.isfinite(w)) and np.all(np.isfinite(v))):
        raise OracleNumericError("eigendecomposition produced non-finite values")
    return Eig(v, w)


def spd_inverse(m: np.ndarray) -> np.ndarray:
    """Lower Cholesky, solve against I, symmetrize (numerics.py:100-114)."""
    n = m.shape[0]
    try:
        factor = scipy.linalg.cho_factor(m, lower=True)
        inv = scipy.linalg.cho_solve(factor, np.eye(n))
    except (np.linalg.LinAlgError, ValueError) as exc:
        raise OracleNumericError(
            f"Cholesky inversion failed for a {n}x{n} matrix (not positive definite?)"
        ) from exc
    if not np.all(np.isfinite(inv)):
        raise OracleNumericError(f"inverse of a {n}x{n} matrix has non-finite entries")
    return 0.5 * (inv + inv.T)


# --------------------------------------------------------------------------
# the per-layer arithmetic (reference kfac.py:85-276)


def compute_factors(x: np.ndarray, gam: np.ndarray):
    """A = X X^T / M and G = Gamma Gamma^T / M, symmetrized (kfac.py:85-104)."""
    for label, arr in (("inputs", x), ("gradients", gam)):
        if arr is None or arr.ndim != 2 or arr.shape[1] == 0:
            raise OracleArgumentError(f"captured {label} must be a nonempty d x B matrix")
    m = x.shape[1]
    if gam.shape[1] != m:
        raise OracleArgumentError("capture batch counts differ")
    a = x @ x.T / m
    g = gam @ gam.T / m
    return 0.5 * (a + a.T), 0.5 * (g + g.T)


def update_running_average(st: LayerState, a_new, g_new, xi: float, t: int) -> LayerState:
    """First call assigns copies; later ``xi*new + (1-xi)*old`` (kfac.py:107-125)."""
    if st.initialized:
        if st.a_cov.shape != a_new.shape or st.g_cov.shape != g_new.shape:
            raise OracleShapeError("factor shapes changed between running-average updates")
        st.a_cov = xi * a_new + (1.0 - xi) * st.a_cov
        st.g_cov = xi * g_new + (1.0 - xi) * st.g_cov
    else:
        st.a_cov, st.g_cov = a_new.copy(), g_new.copy()
        st.initialized = True
    st.last_factor_update = t
    return st


def pi_scalar(a: np.ndarray, g: np.ndarray) -> float:
    """sqrt((tr A / d_A) / (tr G / d_G)) on the raw factors (kfac.py:128-137)."""
    tra, trg = float(np.trace(a)), float(np.trace(g))
    if tra <= 0 or trg <= 0:
        raise OracleNumericError(
            f"degenerate factor: traces must be positive, got Tr(A)={tra}, Tr(G)={trg}")
    return math.sqrt((tra / a.shape[0]) / (trg / g.shape[0]))


def damped_inverses(a: np.ndarray, g: np.ndarray, gamma: float):
    """(A + pi sqrt(gamma) I)^-1, (G + sqrt(gamma)/pi I)^-1 (kfac.py:140-155)."""
    pi = pi_scalar(a, g)
    r = math.sqrt(gamma)
    try:
        a_inv = spd_inverse(a + (pi * r) * np.eye(a.shape[0]))
    except OracleNumericError as exc:
        raise OracleNumericError(f"damped input factor A is not invertible: {exc}") from exc
    try:
        g_inv = spd_inverse(g + (r / pi) * np.eye(g.shape[0]))
    except OracleNumericError as exc:
        raise OracleNumericError(f"damped gradient factor G is not invertible: {exc}") from exc
    return a_inv, g_inv


def _grad_shape_ok(grad, dg, da):
    if grad.shape != (dg, da):
        raise OracleShapeError(f"gradient shape {grad.shape} does not match factor dims ({dg}, {da})")


def precondition_inverse(a, g, grad, gamma):
    """G_inv @ grad @ A_inv with freshly damped inverses (kfac.py:165-171)."""
    _grad_shape_ok(grad, g.shape[0], a.shape[0])
    a_inv, g_inv = damped_inverses(a, g, gamma)
    return g_inv @ grad @ a_inv


def precondition_eigen(a_eig: Eig, g_eig: Eig, grad, gamma):
    """Rotate, divide by clamp(v_g) clamp(v_a)^T + gamma, rotate back (kfac.py:174-191)."""
    _grad_shape_ok(grad, g_eig.q.shape[0], a_eig.q.shape[0])
    denom = np.outer(np.maximum(g_eig.values, 0.0), np.maximum(a_eig.values, 0.0)) + gamma
    if denom.min() <= 0.0:
        raise OracleNumericError(
            f"eigen damping denominator is not positive (min {denom.min()}); "
            "use gamma > 0 or nonsingular factors")
    inner = (g_eig.q.T @ grad @ a_eig.q) / denom
    return g_eig.q @ inner @ a_eig.q.T


def refresh_inverses(st: LayerState, h: Hyper, t: int) -> LayerState:
    """Recompute the held decomposition kind, drop the other (kfac.py:224-241)."""
    if not st.initialized:
        raise OracleOrderingError("cannot build a preconditioner before any factor update")
    if h.inv_type == "eigen":
        st.a_eig, st.g_eig = symmetric_eig(st.a_cov), symmetric_eig(st.g_cov)
        st.a_damped_inv = st.g_damped_inv = None
    else:
        st.a_damped_inv, st.g_damped_inv = damped_inverses(st.a_cov, st.g_cov, h.gamma)
        st.a_eig = st.g_eig = None
    st.last_inverse_update = t
    return st


def apply_preconditioner(st: LayerState, grad, h: Hyper):
    """Use whatever (possibly stale) decomposition is held (kfac.py:244-254)."""
    if h.inv_type == "eigen":
        if st.a_eig is None or st.g_eig is None:
            raise OracleOrderingError("preconditioning requested before any eigendecomposition exists")
        return precondition_eigen(st.a_eig, st.g_eig, grad, h.gamma)
    if st.a_damped_inv is None or st.g_damped_inv is None:
        raise OracleOrderingError("preconditioning requested before any damped inverse exists")
    _grad_shape_ok(grad, st.g_damped_inv.shape[0], st.a_damped_inv.shape[0])
    return st.g_damped_inv @ grad @ st.a_damped_inv


def kfac_layer_step(st: LayerState, x, gam, grad, h: Hyper, t: int):
    """Factor update if due, refresh if due, always precondition (kfac.py:257-276)."""
    if factor_due(t, h):
        a_new, g_new = compute_factors(x, gam)
        update_running_average(st, a_new, g_new, h.xi, t)
    if inverse_due(t, h):
        refresh_inverses(st, h, t)
    return apply_preconditioner(st, grad, h), st


# --------------------------------------------------------------------------
# partition (reference costmodel.py:66-70, distsim.py:86-101)


def round_robin_partition(n_layers: int, workers: int):
    """Worker p owns layers p, p+P, p+2P, ... (costmodel.py:66-70)."""
    if n_layers < 0 or workers < 1:
        raise OracleArgumentError("need n_items >= 0 and n_workers >= 1")
    return tuple(tuple(range(p, n_layers, workers)) for p in range(workers))


def validate_partition(parts, n_layers: int) -> None:
    """Every layer exactly once (distsim.py:93-101)."""
    seen = set()
    for part in parts:
        for i in part:
            if i in seen:
                raise OracleArgumentError(f"layer {i} assigned to more than one worker")
            seen.add(i)
    if seen != set(range(n_layers)):
        raise OracleArgumentError(f"assignment does not cover layers 0..{n_layers - 1} exactly")


# --------------------------------------------------------------------------
# conv linear form (defined by this build at the boundary)


def _pair(v):
    return (int(v[0]), int(v[1])) if isinstance(v, (tuple, list)) else (int(v), int(v))


def unfold_columns(x_nchw: np.ndarray, kh: int, kw: int, stride, pad,
                   dilation=1, bias: bool = False) -> np.ndarray:
    """im2col of an NCHW batch into the reference's column-per-sample form.

    Row order (C_in, kh, kw) == ``weight.view(C_out, -1)`` == ``F.unfold``;
    columns enumerate (n, oh, ow); a ones row is appended LAST when the layer
    has a bias (reference model.py:140-143).  ``stride``, ``pad`` and
    ``dilation`` are ints or (h, w) pairs (Inception's 1x7 / 7x1 convs pad
    (0, 3) / (3, 0)).
    """
    (sh, sw), (ph, pw), (dh, dw) = _pair(stride), _pair(pad), _pair(dilation)
    n, c, h, w = x_nchw.shape
    oh = (h + 2 * ph - dh * (kh - 1) - 1) // sh + 1
    ow = (w + 2 * pw - dw * (kw - 1) - 1) // sw + 1
    xp = np.zeros((n, c, h + 2 * ph, w + 2 * pw), dtype=np.float64)
    xp[:, :, ph:ph + h, pw:pw + w] = x_nchw
    cols = np.empty((c, kh, kw, n, oh, ow), dtype=np.float64)
    for i in range(kh):
        for j in range(kw):
            hs, ws = i * dh, j * dw
            cols[:, i, j] = xp[:, :, hs:hs + sh * oh:sh, ws:ws + sw * ow:sw].transpose(1, 0, 2, 3)
    out = cols.reshape(c * kh * kw, n * oh * ow)
    if bias:
        out = np.vstack([out, np.ones((1, out.shape[1]))])
    return out
