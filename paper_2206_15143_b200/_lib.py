"""ctypes binding of libdpkfac.so (the C ABI declared in include/dpkfac.h).

The structures below mirror the C structs field for field; ``tests/test_abi.py``
checks their sizes against the header.  Loading fails loudly when the shared
library is missing -- there is no CPU or eager fallback anywhere in the package.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DPK_LIB_PATH") or os.path.join(_HERE, "libdpkfac.so")  # override: experiments only

DPK_OK, DPK_EARG, DPK_ESHAPE, DPK_ECUDA, DPK_ENOSPACE = 0, 1, 2, 3, 4
DPK_PREC_TF32, DPK_PREC_TF32_TRUNC, DPK_PREC_3XTF32, DPK_PREC_3XF16 = 1, 2, 3, 4
INFO_OK, INFO_TRACE, INFO_NOT_SPD_A, INFO_NOT_SPD_G, INFO_EIG_DENOM, INFO_NONFINITE = range(6)
OPND_ROWS_K, OPND_ROWS_MN, OPND_IM2COL, OPND_IM2COL_TAPMAJOR, OPND_ROWS_K_F16, OPND_IM2COL_TAPMAJOR_F16 = 0, 1, 2, 3, 4, 5


class Operand(C.Structure):
    _fields_ = [
        ("data", C.c_void_p),
        ("kind", C.c_int32), ("rows", C.c_int32), ("bias_row", C.c_int32), ("_pad0", C.c_int32),
        ("cols", C.c_int64), ("ld", C.c_int64),
        ("C", C.c_int32), ("H", C.c_int32), ("W", C.c_int32), ("OH", C.c_int32), ("OW", C.c_int32),
        ("kh", C.c_int32), ("kw", C.c_int32), ("sh", C.c_int32), ("sw", C.c_int32),
        ("ph", C.c_int32), ("pw", C.c_int32), ("dh", C.c_int32), ("dw", C.c_int32),
        ("_pad1", C.c_int32),
        ("sn", C.c_int64), ("sc", C.c_int64), ("shs", C.c_int64), ("sws", C.c_int64),
    ]


class FactorJob(C.Structure):
    _fields_ = [("x", Operand), ("factor", C.c_void_p), ("alpha", C.c_float), ("beta", C.c_float),
                ("x_amax", C.c_void_p)]


class Im2colJob(C.Structure):
    _fields_ = [("x", Operand), ("out", C.c_void_p), ("ld", C.c_int64), ("amax", C.c_void_p)]


class GemmJob(C.Structure):
    _fields_ = [
        ("a", Operand), ("b", Operand),
        ("out", C.c_void_p), ("ldo", C.c_int64),
        ("cin", C.c_void_p), ("ldc", C.c_int64),
        ("alpha", C.c_float), ("beta", C.c_float),
        ("symmetric", C.c_int32), ("_pad0", C.c_int32),
    ]


class PiJob(C.Structure):
    _fields_ = [("a", C.c_void_p), ("g", C.c_void_p), ("da", C.c_int32), ("dg", C.c_int32),
                ("shifts", C.c_void_p), ("pi", C.c_void_p), ("info", C.c_void_p)]


class SpdJob(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("n", C.c_int32), ("fail_code", C.c_int32),
                ("shift", C.c_void_p), ("info", C.c_void_p)]


class SpdFactorJob(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("ldd", C.c_int64), ("n", C.c_int32),
                ("fail_code", C.c_int32), ("shift", C.c_void_p), ("info", C.c_void_p)]


class PrecondFactorJob(C.Structure):
    _fields_ = [("grad", C.c_void_p), ("xa", C.c_void_p), ("xg", C.c_void_p), ("out", C.c_void_p),
                ("tmp", C.c_void_p), ("ldxa", C.c_int64), ("ldxg", C.c_int64),
                ("d_out", C.c_int32), ("d_in", C.c_int32)]


class PrecondJob(C.Structure):
    _fields_ = [("grad", C.c_void_p), ("a_mat", C.c_void_p), ("g_mat", C.c_void_p),
                ("a_vals", C.c_void_p), ("g_vals", C.c_void_p), ("out", C.c_void_p), ("tmp", C.c_void_p),
                ("d_out", C.c_int32), ("d_in", C.c_int32), ("info", C.c_void_p)]


class EigJob(C.Structure):
    _fields_ = [("src", C.c_void_p), ("q", C.c_void_p), ("w", C.c_void_p), ("n", C.c_int32),
                ("_pad0", C.c_int32), ("info", C.c_void_p)]


class Segment(C.Structure):
    _fields_ = [("weight", C.c_void_p), ("bias", C.c_void_p), ("offset", C.c_int64),
                ("rows", C.c_int32), ("cols_w", C.c_int32), ("ldw", C.c_int64),
                ("perm_khw", C.c_int32), ("_pad0", C.c_int32)]


# every exported symbol of include/dpkfac.h: (name, restype, argtypes)
_P = C.c_void_p
_SIGNATURES = [
    ("dpk_factor_workspace_bytes", C.c_size_t, [C.POINTER(FactorJob), C.c_int]),
    ("dpk_syrk_ema", C.c_int, [C.POINTER(FactorJob), C.c_int, _P, C.c_size_t, C.c_int, _P]),
    ("dpk_conv_im2col_syrk_ema", C.c_int, [C.POINTER(FactorJob), C.c_int, _P, C.c_size_t, C.c_int, _P]),
    ("dpk_im2col_materialize", C.c_int, [C.POINTER(Im2colJob), C.c_int, _P]),
    ("dpk_im2col_materialize_f16", C.c_int, [C.POINTER(Im2colJob), C.c_int, _P]),
    ("dpk_im2col_amax", C.c_int, [C.POINTER(Im2colJob), C.c_int, _P]),
    ("dpk_im2col_convert_f16", C.c_int, [C.POINTER(Im2colJob), C.c_int, _P]),
    ("dpk_gemm_workspace_bytes", C.c_size_t, [C.POINTER(GemmJob), C.c_int]),
    ("dpk_gemm", C.c_int, [C.POINTER(GemmJob), C.c_int, _P, C.c_size_t, C.c_int, _P]),
    ("dpk_trace_pi", C.c_int, [C.POINTER(PiJob), C.c_int, C.c_float, _P]),
    ("dpk_chol_inv_workspace_bytes", C.c_size_t, [C.POINTER(SpdJob), C.c_int]),
    ("dpk_chol_inv_damped_batched", C.c_int, [C.POINTER(SpdJob), C.c_int, _P, C.c_size_t, _P]),
    ("dpk_chol_factor_inv_workspace_bytes", C.c_size_t, [C.POINTER(SpdFactorJob), C.c_int]),
    ("dpk_chol_factor_inv_batched", C.c_int, [C.POINTER(SpdFactorJob), C.c_int, _P, C.c_size_t, _P]),
    ("dpk_precond_factor_workspace_bytes", C.c_size_t, [C.POINTER(PrecondFactorJob), C.c_int]),
    ("dpk_precond_factored", C.c_int, [C.POINTER(PrecondFactorJob), C.c_int, _P, C.c_size_t, C.c_int, _P]),
    ("dpk_precond_workspace_bytes", C.c_size_t, [C.POINTER(PrecondJob), C.c_int]),
    ("dpk_precond_inverse", C.c_int, [C.POINTER(PrecondJob), C.c_int, _P, C.c_size_t, C.c_int, _P]),
    ("dpk_precond_eigen", C.c_int, [C.POINTER(PrecondJob), C.c_int, C.c_float, _P, C.c_size_t, C.c_int, _P]),
    ("dpk_syevd_workspace_bytes", C.c_size_t, [C.POINTER(EigJob), C.c_int]),
    ("dpk_syevd_batched", C.c_int, [C.POINTER(EigJob), C.c_int, _P, C.c_size_t, _P]),
    ("dpk_pack_owner_major", C.c_int, [C.POINTER(Segment), C.c_int, _P, C.c_float, _P]),
    ("dpk_unpack_owner_major", C.c_int, [C.POINTER(Segment), C.c_int, _P, C.c_float, _P]),
    ("dpk_kl_dot_workspace_bytes", C.c_size_t, []),
    ("dpk_kl_dot", C.c_int, [_P, _P, C.c_int64, _P, _P, C.c_size_t, _P]),
    ("dpk_unpack_owner_major_klclip", C.c_int, [C.POINTER(Segment), C.c_int, _P, C.c_float, _P, C.c_int,
                                                C.c_int64, C.c_float, C.c_float, _P]),
    ("dpk_ipc_export", C.c_int, [_P, C.c_int, _P, C.POINTER(C.c_int64)]),
    ("dpk_ipc_open", C.c_int, [_P, C.c_int, C.POINTER(C.c_void_p)]),
    ("dpk_ipc_close", C.c_int, [_P]),
    ("dpk_peer_gather", C.c_int, [_P, C.POINTER(C.c_void_p), C.c_int, C.c_int64, _P]),
    ("dpk_version", C.c_char_p, []),
    ("dpk_last_error", C.c_char_p, []),
    ("dpk_launch_count", C.c_ulonglong, []),
    ("dpk_debug_timestamps", C.c_int, [C.POINTER(C.c_ulonglong)]),
    ("dpk_debug_unit_timestamps", C.c_int, [C.POINTER(C.c_ulonglong)]),
    ("dpk_set_launch_cap", C.c_int, [C.c_int]),
]

EXPORTED = tuple(name for name, _, _ in _SIGNATURES)

_lib = None


class LibraryMissing(ImportError):
    pass


def load(path: str = LIB_PATH):
    """Load libdpkfac.so once; raise (never fall back) if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryMissing(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, res, args in _SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def array(struct_type, items):
    arr = (struct_type * max(len(items), 1))()
    for i, it in enumerate(items):
        arr[i] = it
    return arr


def check(rc: int, what: str):
    if rc == DPK_OK:
        return
    from .errors import ArgumentError, KfacLabError, ShapeError
    msg = f"{what}: {_lib.dpk_last_error().decode(errors='replace')}"
    if rc == DPK_EARG:
        raise ArgumentError(msg)
    if rc == DPK_ESHAPE:
        raise ShapeError(msg)
    raise KfacLabError(f"{msg} (code {rc})")
