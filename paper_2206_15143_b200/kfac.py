"""Functional K-FAC surface on CUDA tensors, mirroring kfaclab kfac.py / numerics.py.

Same function names, argument meanings, return conventions and error classes
as the reference (kfac.py:39-276, numerics.py:75-114); the arithmetic runs in
libdpkfac.so on the GPU in float32 (factors on tcgen05 TF32, inverses with
3xTF32 recursion, preconditioning on tcgen05).  These functions are the parity
surface the tests drive against the float64 oracle; the DP-KFAC optimizer
(``DPKFAC``) calls the same kernels in grouped launches.

Layouts follow the reference: captures are d x M (columns = samples), factors
d x d, gradients d_out x d_in.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple, Optional

import torch

from . import _lib as L
from . import ops
from .errors import ArgumentError, NumericError, OrderingError, ShapeError

INV_TYPES = ("inverse", "eigen")


class EigenPair(NamedTuple):
    """Orthonormal eigenvectors (columns of ``q``) and descending eigenvalues (numerics.py:33-37)."""

    q: torch.Tensor
    values: torch.Tensor


@dataclass(frozen=True)
class KfacHyper:
    """Damping gamma, running-average weight xi (weights the NEW factor),
    damping scheme, factor / inverse refresh intervals (kfac.py:55-74)."""

    gamma: float = 0.03
    xi: float = 0.95
    inv_type: str = "eigen"
    f_freq: int = 1
    k_freq: int = 1

    def __post_init__(self):
        if self.gamma < 0:
            raise ArgumentError("damping gamma must be >= 0")
        if not (0.0 < self.xi <= 1.0):
            raise ArgumentError("running-average weight xi must lie in (0, 1]")
        if self.inv_type not in INV_TYPES:
            raise ArgumentError(f"inv_type must be one of {INV_TYPES}")
        if self.f_freq < 1 or self.k_freq < 1:
            raise ArgumentError("f_freq and k_freq must be >= 1")


@dataclass
class FactorState:
    """Per-layer curvature state (kfac.py:39-52), device-resident."""

    a_cov: Optional[torch.Tensor] = None
    g_cov: Optional[torch.Tensor] = None
    a_eig: Optional[EigenPair] = None
    g_eig: Optional[EigenPair] = None
    a_damped_inv: Optional[torch.Tensor] = None
    g_damped_inv: Optional[torch.Tensor] = None
    last_factor_update: int = -1
    last_inverse_update: int = -1
    initialized: bool = False


def is_factor_update(t: int, hyper: KfacHyper) -> bool:
    return t % hyper.f_freq == 0


def is_inverse_update(t: int, hyper: KfacHyper) -> bool:
    return t % hyper.k_freq == 0


def _f32(x) -> torch.Tensor:
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise ArgumentError("expected a CUDA tensor")
    return x.float().contiguous()


def _square(m: torch.Tensor, name: str) -> torch.Tensor:
    if m.dim() != 2 or m.shape[0] != m.shape[1]:
        raise ShapeError(f"{name}: expected a square matrix, got {tuple(m.shape)}")
    return m


def _raise_info(code: int, n: int, side: str = "") -> None:
    if code == L.INFO_OK:
        return
    if code == L.INFO_TRACE:
        raise NumericError("degenerate factor: traces must be positive")
    if code in (L.INFO_NOT_SPD_A, L.INFO_NOT_SPD_G):
        which = "damped input factor A" if code == L.INFO_NOT_SPD_A else "damped gradient factor G"
        raise NumericError(f"{which} is not invertible: Cholesky inversion failed for a {n}x{n} matrix "
                           "(not positive definite?)")
    if code == L.INFO_EIG_DENOM:
        raise NumericError("eigen damping denominator is not positive; use gamma > 0 or nonsingular factors")
    raise NumericError(f"eigendecomposition produced non-finite values for a {n}x{n} matrix")


# ------------------------------------------------------------------ numerics.py
def sym_eig(m: torch.Tensor, solver: str = "cusolver") -> EigenPair:
    """Symmetrize, decompose, descending order (numerics.py:75-97).  n > 128:
    ``solver`` "cusolver" (default) or "native" (tensor-core block Jacobi)."""
    m = _square(_f32(m), "sym_eig")
    n = m.shape[0]
    q = torch.empty_like(m)
    w = torch.empty(n, device=m.device, dtype=torch.float32)
    info = torch.zeros(1, dtype=torch.int32, device=m.device)
    ops.syevd([(m, q, w, info)], solver)
    _raise_info(int(info.item()), n)
    return EigenPair(q, w)


def sym_inverse(m: torch.Tensor) -> torch.Tensor:
    """Inverse of an SPD matrix, exactly symmetric (numerics.py:100-114)."""
    m = _square(_f32(m), "sym_inverse")
    n = m.shape[0]
    out = torch.empty_like(m)
    info = torch.zeros(1, dtype=torch.int32, device=m.device)
    ops.chol_inv([ops.spd_job(m, out, None, info, L.INFO_NOT_SPD_A)])
    if int(info.item()) != 0:
        raise NumericError(f"Cholesky inversion failed for a {n}x{n} matrix (not positive definite?)")
    return out


# ------------------------------------------------------------------ kfac.py
def _check_captures(captured_inputs, captured_preact_grads):
    for name, arr in (("inputs", captured_inputs), ("gradients", captured_preact_grads)):
        if arr is None or arr.dim() != 2 or arr.shape[1] == 0:
            raise ArgumentError(f"captured {name} must be a nonempty d x B matrix")
    batch = captured_inputs.shape[1]
    if captured_preact_grads.shape[1] != batch:
        raise ArgumentError(f"capture batch counts differ: {batch} inputs vs "
                            f"{captured_preact_grads.shape[1]} gradients")


def compute_factors(captured_inputs: torch.Tensor, captured_preact_grads: torch.Tensor,
                    precision: str = "tf32") -> tuple[torch.Tensor, torch.Tensor]:
    """A = X X^T / M, G = Gamma Gamma^T / M, exactly symmetric (kfac.py:85-104)."""
    _check_captures(captured_inputs, captured_preact_grads)
    x, g = _f32(captured_inputs), _f32(captured_preact_grads)
    m = x.shape[1]
    a_new = torch.empty(x.shape[0], x.shape[0], device=x.device)
    g_new = torch.empty(g.shape[0], g.shape[0], device=x.device)
    ops.syrk_ema([ops.factor_job(ops.operand_rows_k(x), a_new, 1.0 / m, 0.0),
                  ops.factor_job(ops.operand_rows_k(g), g_new, 1.0 / m, 0.0)], precision)
    return a_new, g_new


def compute_conv_input_factor(x: torch.Tensor, kernel_size, stride=1, padding=0, dilation=1, bias: bool = False,
                              precision: str = "3xtf32") -> torch.Tensor:
    """A = X X^T / M for a Conv2d input x (N x C x H x W, NCHW or channels-last) without
    materializing X: X is the conv's implicit-im2col linear form -- rows in the
    reference (C, kh, kw) = ``weight.view(C_out, -1)`` order, columns (n, oh, ow), a
    ones row last when the layer has a bias (kfac.py:85-104
    applied to ``F.unfold`` columns).  One ``dpk_conv_im2col_syrk_ema`` launch."""
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dim() != 4:
        raise ArgumentError("expected a 4-D CUDA conv input")
    pair = lambda v: (int(v[0]), int(v[1])) if isinstance(v, (tuple, list)) else (int(v), int(v))
    x = x.float()
    op = ops.operand_im2col(x, pair(kernel_size), pair(stride), pair(padding), pair(dilation), bias_row=bias)
    if op.cols < 1:
        raise ArgumentError("captured inputs must be a nonempty d x B matrix")
    d = op.rows + op.bias_row
    a = torch.empty(d, d, device=x.device)
    ops.conv_syrk_ema([ops.factor_job(op, a, 1.0 / op.cols, 0.0)], precision)
    return a


def update_running_average(state: FactorState, a_new, g_new, xi: float, t: int) -> FactorState:
    """First update assigns copies; later xi*new + (1-xi)*old (kfac.py:107-125)."""
    if not state.initialized:
        state.a_cov = a_new.clone()
        state.g_cov = g_new.clone()
        state.initialized = True
    else:
        if state.a_cov.shape != a_new.shape or state.g_cov.shape != g_new.shape:
            raise ShapeError("factor shapes changed between running-average updates")
        state.a_cov = xi * a_new + (1.0 - xi) * state.a_cov
        state.g_cov = xi * g_new + (1.0 - xi) * state.g_cov
    state.last_factor_update = t
    return state


def update_factors_fused(state: FactorState, captured_inputs, captured_preact_grads, xi: float, t: int,
                         precision: str = "tf32") -> FactorState:
    """compute_factors + update_running_average in ONE tensor-core launch: the
    EMA is the SYRK epilogue (alpha = xi/M, beta = 1 - xi; first update assigns)."""
    _check_captures(captured_inputs, captured_preact_grads)
    x, g = _f32(captured_inputs), _f32(captured_preact_grads)
    m = x.shape[1]
    first = not state.initialized
    if first:
        state.a_cov = torch.empty(x.shape[0], x.shape[0], device=x.device)
        state.g_cov = torch.empty(g.shape[0], g.shape[0], device=x.device)
    elif state.a_cov.shape[0] != x.shape[0] or state.g_cov.shape[0] != g.shape[0]:
        raise ShapeError("factor shapes changed between running-average updates")
    w = 1.0 if first else xi
    beta = 0.0 if first else 1.0 - xi
    ops.syrk_ema([ops.factor_job(ops.operand_rows_k(x), state.a_cov, w / m, beta),
                  ops.factor_job(ops.operand_rows_k(g), state.g_cov, w / m, beta)], precision)
    state.initialized = True
    state.last_factor_update = t
    return state


def pi_scalar(a_cov: torch.Tensor, g_cov: torch.Tensor) -> float:
    """sqrt((tr A / d_A) / (tr G / d_G)) on the raw factors (kfac.py:128-137)."""
    tr_a = float(torch.diagonal(a_cov).double().sum())
    tr_g = float(torch.diagonal(g_cov).double().sum())
    if tr_a <= 0 or tr_g <= 0:
        raise NumericError(f"degenerate factor: traces must be positive, got Tr(A)={tr_a}, Tr(G)={tr_g}")
    return float(math.sqrt((tr_a / a_cov.shape[0]) / (tr_g / g_cov.shape[0])))


def _damped_inverses_device(pairs, gamma: float):
    """Grouped: traces/pi on device, then batched damped inverses.  Returns
    ([(a_inv, g_inv)], info tensor)."""
    dev = pairs[0][0].device
    n = len(pairs)
    shifts = torch.empty(n, 2, device=dev)
    info = torch.zeros(n, dtype=torch.int32, device=dev)
    ops.trace_pi(pairs, gamma, shifts, None, [info[i] for i in range(n)])
    outs, jobs = [], []
    for i, (a, g) in enumerate(pairs):
        ai, gi = torch.empty_like(a), torch.empty_like(g)
        jobs.append(ops.spd_job(a, ai, shifts[i, 0], info[i], L.INFO_NOT_SPD_A))
        jobs.append(ops.spd_job(g, gi, shifts[i, 1], info[i], L.INFO_NOT_SPD_G))
        outs.append((ai, gi))
    ops.chol_inv(jobs)
    return outs, info


def damped_inverses(a_cov: torch.Tensor, g_cov: torch.Tensor, gamma: float):
    """Cholesky-grade inverses of the pi-split damped factors (kfac.py:140-155)."""
    a, g = _square(_f32(a_cov), "A"), _square(_f32(g_cov), "G")
    (res,), info = _damped_inverses_device([(a, g)], gamma)
    code = int(info.item())
    _raise_info(code, a.shape[0] if code != L.INFO_NOT_SPD_G else g.shape[0])
    return res


def _check_grad_shape(grad, dim_g: int, dim_a: int):
    if tuple(grad.shape) != (dim_g, dim_a):
        raise ShapeError(f"gradient shape {tuple(grad.shape)} does not match factor dims ({dim_g}, {dim_a})")


def _precondition(grad, a_mat, g_mat, eigen: bool, gamma: float, a_vals=None, g_vals=None,
                  precision: str = "3xtf32"):
    grad = _f32(grad)
    out = torch.empty_like(grad)
    tmp = torch.empty_like(grad)
    info = torch.zeros(1, dtype=torch.int32, device=grad.device)
    ops.precondition([ops.precond_job(grad, a_mat, g_mat, out, tmp, a_vals, g_vals, info)], eigen, gamma, precision)
    if eigen:
        _raise_info(int(info.item()), 0)
    return out


def precondition_inverse(a_cov, g_cov, grad, gamma: float, precision: str = "3xtf32"):
    """(G + sqrt(g)/pi I)^-1 grad (A + pi sqrt(g) I)^-1 (kfac.py:165-171)."""
    _check_grad_shape(grad, g_cov.shape[0], a_cov.shape[0])
    a_inv, g_inv = damped_inverses(a_cov, g_cov, gamma)
    return _precondition(grad, a_inv, g_inv, False, gamma, precision=precision)


def precondition_eigen(a_eig: EigenPair, g_eig: EigenPair, grad, gamma: float, precision: str = "3xtf32"):
    """Q_G ((Q_G^T grad Q_A) / (max(v_G,0) max(v_A,0)^T + gamma)) Q_A^T (kfac.py:174-191)."""
    _check_grad_shape(grad, g_eig.q.shape[0], a_eig.q.shape[0])
    return _precondition(grad, _f32(a_eig.q), _f32(g_eig.q), True, gamma, _f32(a_eig.values),
                         _f32(g_eig.values), precision)


def refresh_inverses(state: FactorState, hyper: KfacHyper, t: int) -> FactorState:
    """Recompute the decomposition kind the hyper asks for; drop the other (kfac.py:224-241)."""
    if not state.initialized:
        raise OrderingError("cannot build a preconditioner before any factor update")
    if hyper.inv_type == "eigen":
        state.a_eig = sym_eig(state.a_cov)
        state.g_eig = sym_eig(state.g_cov)
        state.a_damped_inv = None
        state.g_damped_inv = None
    else:
        state.a_damped_inv, state.g_damped_inv = damped_inverses(state.a_cov, state.g_cov, hyper.gamma)
        state.a_eig = None
        state.g_eig = None
    state.last_inverse_update = t
    return state


def apply_preconditioner(state: FactorState, grad, hyper: KfacHyper, precision: str = "3xtf32"):
    """Precondition with the (possibly stale) held decomposition (kfac.py:244-254)."""
    if hyper.inv_type == "eigen":
        if state.a_eig is None or state.g_eig is None:
            raise OrderingError("preconditioning requested before any eigendecomposition exists")
        return precondition_eigen(state.a_eig, state.g_eig, grad, hyper.gamma, precision)
    if state.a_damped_inv is None or state.g_damped_inv is None:
        raise OrderingError("preconditioning requested before any damped inverse exists")
    _check_grad_shape(grad, state.g_damped_inv.shape[0], state.a_damped_inv.shape[0])
    return _precondition(grad, state.a_damped_inv, state.g_damped_inv, False, hyper.gamma, precision=precision)


def kfac_layer_step(state: FactorState, captured_inputs, captured_preact_grads, grad, hyper: KfacHyper, t: int,
                    precision: str = "auto", precond_precision: str = "3xtf32"):
    """Factor update if due (fused SYRK+EMA), refresh if due, always precondition
    (kfac.py:257-276).  Returns (preconditioned grad, state).  ``precision``
    applies to the factor SYRK ("auto": 3xtf32 for eigen, tf32 for inverse -- the
    same rule as DPKFAC), ``precond_precision`` to the preconditioning GEMMs."""
    if precision == "auto":
        precision = "3xtf32" if hyper.inv_type == "eigen" else "tf32"
    if is_factor_update(t, hyper):
        update_factors_fused(state, captured_inputs, captured_preact_grads, hyper.xi, t, precision)
    if is_inverse_update(t, hyper):
        refresh_inverses(state, hyper, t)
    return apply_preconditioner(state, grad, hyper, precond_precision), state
