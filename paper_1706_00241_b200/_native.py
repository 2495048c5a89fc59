"""ctypes binding of ``libdefcg_b200.so`` (C ABI in include/defcg_b200.h).

There is deliberately no fallback: if the library is missing or no CUDA device
is present, every call raises (``ImportError`` / ``DeviceError``), so a test or
benchmark can never pass on a silent CPU path.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import (
    BasisDeficient,
    BreakdownZeroCurvature,
    DeviceError,
    DimensionMismatch,
    GramNotSpd,
    NoConvergence,
    NotPositiveDefinite,
)

# DCG_LIB_PATH: a developer build of the same library (e.g. a variant with
# different compile-time tuning, ``python -m paper_1706_00241_b200.build
# --variant DIR -DNAME=VALUE``); the in-tree build otherwise.
LIB_PATH = Path(os.environ.get("DCG_LIB_PATH") or Path(__file__).resolve().with_name("libdefcg_b200.so"))

DCG_OK = 0
DCG_E_DIMENSION = 1
DCG_E_NOT_PD = 2
DCG_E_BREAKDOWN = 3
DCG_E_GRAM_NOT_SPD = 4
DCG_E_BASIS_DEFICIENT = 5
DCG_E_NO_CONVERGENCE = 6
DCG_E_ASYMMETRIC = 7
DCG_E_CONFIG = 8
DCG_E_CUDA = 9
DCG_E_UNSUPPORTED = 10

DCG_OP_DENSE = 0
DCG_OP_RBF = 1
DCG_OP_DENSE_SYM = 2
DCG_SELECT_SMALLEST = 0
DCG_SELECT_LARGEST = 1
MAX_K = 64
MAX_T = 112

_P = ctypes.c_void_p
_LL = ctypes.c_longlong
_D = ctypes.c_double
_PLL = ctypes.POINTER(ctypes.c_longlong)
_PD = ctypes.POINTER(ctypes.c_double)
_PI = ctypes.POINTER(ctypes.c_int)


class COperator(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("n", _LL),
        ("row0", _LL),
        ("rows", _LL),
        ("d_k", _P),
        ("ldk", _LL),
        ("d_x", _P),
        ("dim", _LL),
        ("var", _D),
        ("inv_two_ell2", _D),
        ("diag", _D),
        ("d_s", _P),
        ("shift", _D),
        ("d_kp", _P),
    ]


class CBasis(ctypes.Structure):
    _fields_ = [("k", _LL), ("d_w", _P), ("d_aw", _P), ("d_chol", _P)]


class CSolverConfig(ctypes.Structure):
    _fields_ = [("tol", _D), ("max_iters", _LL), ("ell", _LL), ("recompute_residual_every", _LL)]


class CKrylovLog(ctypes.Structure):
    _fields_ = [
        ("ell", _LL),
        ("d_p", _P),
        ("d_r", _P),
        ("d_d", _P),
        ("d_alpha", _P),
        ("d_beta", _P),
        ("d_mu", _P),
    ]


class CSolveInfo(ctypes.Structure):
    _fields_ = [
        ("iterations", _LL),
        ("stored", _LL),
        ("converged", ctypes.c_int),
        ("termination", ctypes.c_int),
        ("rel_residual", _D),
        ("norm_b", _D),
        ("device_ms", _D),
    ]


_RESTYPES = {"dcg_status_string": ctypes.c_char_p, "dcg_launch_count": ctypes.c_longlong,
             "dcg_packed_sym_doubles": ctypes.c_longlong}

# name -> argtypes (restype is always c_int unless listed in _RESTYPES)
SIGNATURES = {
    "dcg_version": [],
    "dcg_launch_count": [],
    "dcg_status_string": [ctypes.c_int],
    "dcg_context_create": [ctypes.c_int, ctypes.POINTER(_P)],
    "dcg_context_destroy": [_P],
    "dcg_context_grid": [_P, _PI, _PI],
    "dcg_k_matvec": [_P, _P, _P, _LL, _LL, _LL, _P, _P],
    "dcg_k_gemm": [_P, _P, _P, _P, _P, _LL, _LL, _LL],
    "dcg_k_cholesky": [_P, _P, _P, _LL, _D, _P, _PLL],
    "dcg_k_solve_lower": [_P, _P, _P, _LL, _P, _P],
    "dcg_k_solve_lower_trans": [_P, _P, _P, _LL, _P, _P],
    "dcg_k_rbf_gram": [_P, _P, _P, _LL, _LL, _D, _D, _D, _P, _LL, _LL, _LL],
    "dcg_k_rbf_cross": [_P, _P, _P, _LL, _P, _LL, _LL, _D, _D, _P],
    "dcg_k_jacobi_sweep": [_P, _P, _P, _P, _LL, _PLL],
    "dcg_check_symmetric": [_P, _P, _P, _LL, _LL, _D, _PI],
    "dcg_packed_sym_doubles": [_LL],
    "dcg_gpc_init": [_P, _P, _LL, _P, _P, _P, _P, _P, ctypes.POINTER(_D), _PLL],
    "dcg_gpc_init_async": [_P, _P, _LL, _P, _P, _P, _P, _P, _P],
    "dcg_block_uses_packed": [ctypes.c_int],
    "dcg_pack_sym": [_P, _P, _P, _LL, _LL, _P],
    "dcg_sym_eigen": [_P, _P, _P, _LL, _LL, _D, _P, _P, _PLL],
    "dcg_gen_sym_eigen": [_P, _P, _P, _P, _LL, _LL, _P, _P, _PLL],
    "dcg_op_apply": [_P, _P, ctypes.POINTER(COperator), _P, _P],
    "dcg_op_apply_block": [_P, _P, ctypes.POINTER(COperator), _P, _LL, _P],
    "dcg_gram_factor": [_P, _P, _P, _P, _LL, _LL, ctypes.c_int, _P, _PLL, _PLL],
    "dcg_refresh_basis": [_P, _P, ctypes.POINTER(COperator), _P, _LL, _P, _P, _P, _PLL, _PLL],
    "dcg_solve": [
        _P,
        _P,
        ctypes.POINTER(COperator),
        _P,
        _P,
        ctypes.POINTER(CBasis),
        ctypes.POINTER(CSolverConfig),
        _P,
        ctypes.POINTER(CKrylovLog),
        _P,
        ctypes.POINTER(CSolveInfo),
        _PLL,
    ],
    "dcg_solve_async": [
        _P,
        _P,
        ctypes.POINTER(COperator),
        _P,
        _P,
        ctypes.POINTER(CBasis),
        ctypes.POINTER(CSolverConfig),
        _P,
        ctypes.POINTER(CKrylovLog),
        _P,
        _P,
        _P,
        _P,
    ],
    "dcg_refresh_basis_async": [_P, _P, ctypes.POINTER(COperator), _P, _LL, _P, _P, _P, _P, _P],
    "dcg_deflation_project": [_P, _P, _LL, ctypes.POINTER(CBasis), _P, _P],
    "dcg_ritz_extract": [
        _P,
        _P,
        _LL,
        ctypes.POINTER(CKrylovLog),
        _LL,
        ctypes.POINTER(CBasis),
        _LL,
        ctypes.c_int,
        _P,
        _P,
        _P,
        _P,
        _P,
        _PLL,
        _PLL,
    ],
    "dcg_ritz_extract_async": [
        _P,
        _P,
        _LL,
        ctypes.POINTER(CKrylovLog),
        _LL,
        ctypes.POINTER(CBasis),
        _LL,
        ctypes.c_int,
        _P,
        _P,
        _P,
        _P,
        _P,
        _P,
    ],
    "dcg_ritz_extract_dev": [
        _P,
        _P,
        _LL,
        ctypes.POINTER(CKrylovLog),
        _P,
        ctypes.POINTER(CBasis),
        _LL,
        ctypes.c_int,
        _P,
        _P,
        _P,
        _P,
        ctypes.c_int,
    ],
    "dcg_gpc_derivs": [_P, _P, _LL, _P, _P, _P, _P, _PD],
    "dcg_gpc_newton_system": [_P, _P, ctypes.POINTER(COperator), _P, _P, _P, _P, _P, _P],
    "dcg_gpc_newton_system_ax0": [_P, _P, ctypes.POINTER(COperator), _P, _P, _P, _P, _P, _P, _P, _P],
    "dcg_gpc_newton_update": [_P, _P, ctypes.POINTER(COperator), _P, _P, _P, _P, _P, _P, _P, _P, _PD, _PD],
    "dcg_gpc_objective": [_P, _P, _LL, _P, _P, _P, _P, _P, _PD, _PD],
    "dcg_gpc_newton_update_async": [_P, _P, ctypes.POINTER(COperator), _P, _P, _P, _P, _P, _P, _P, _P, _P],
    # row-sharded def-CG (include/defcg_b200.h L5)
    "dcg_shard_apply_dot": [_P, _P, ctypes.POINTER(COperator), _P, _P, _P, _P],
    "dcg_shard_rbf_sym_partial": [_P, _P, ctypes.POINTER(COperator), ctypes.c_int, ctypes.c_int, _P, _P, _P],
    "dcg_shard_tile_range": [_LL, ctypes.c_int, ctypes.c_int, _PLL, _PLL],
    "dcg_shard_start_r": [_P, _P, _LL, ctypes.c_int, _P, _P, _P, _P, _P, _P, _P, _P, _D, _LL, _LL],
    "dcg_k_rbf_gram_packed": [_P, _P, _P, _LL, _LL, _D, _D, _D, _LL, _LL, _P],
    "dcg_shard_tiles_partial": [_P, _P, ctypes.POINTER(COperator), ctypes.c_int, ctypes.c_int, _P, _P, _P],
    "dcg_shard_tiles_partial2": [_P, _P, ctypes.POINTER(COperator), ctypes.c_int, ctypes.c_int, _P, _P, _P, _P],
    "dcg_shard_epilogue": [_P, _P, ctypes.c_int, ctypes.POINTER(COperator), _P, _P, _P, _P, _P, _P],
    "dcg_shard_residual": [_P, _P, ctypes.POINTER(COperator), _P, _P, _P, _P],
    "dcg_shard_partials": [_P, _P, _LL, ctypes.c_int, _P, _P, _P, _P],
    "dcg_shard_start": [_P, _P, _LL, ctypes.c_int, _P, _P, _P, _P, _P, _P, _D, _LL, _LL],
    "dcg_shard_begin": [_P, _P, _LL, ctypes.c_int, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "dcg_shard_update": [_P, _P, ctypes.c_int, _LL, ctypes.c_int, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "dcg_shard_direction": [_P, _P, _LL, ctypes.c_int, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "dcg_shard_step": [_P, _P, _LL, ctypes.c_int, _P, _P, ctypes.c_double, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                       _P, _P, _P, _P],
}

# dcg_shard_state (include/defcg_b200.h): 7 doubles then 9 int64, 128 bytes
SHARD_STATE_DOUBLES = 16
SHARD_RR, SHARD_NORM_B, SHARD_REL, SHARD_ALPHA, SHARD_BETA, SHARD_D, SHARD_TOL = range(7)
SHARD_IT, SHARD_MAX_ITERS, SHARD_DONE, SHARD_STATUS, SHARD_INFO, SHARD_ELL = range(7, 13)

_lib = None
_lock = threading.Lock()
_contexts: dict[tuple[int, int], int] = {}


def load_library():
    """Load the CUDA library (ImportError, never a fallback, when absent)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise ImportError(
                        f"{LIB_PATH.name} is not built (run `python -m paper_1706_00241_b200.build`); "
                        "the def-CG path has no CPU fallback"
                    )
                lib = ctypes.CDLL(str(LIB_PATH))
                for name, args in SIGNATURES.items():
                    fn = getattr(lib, name)
                    fn.argtypes = args
                    fn.restype = _RESTYPES.get(name, ctypes.c_int)
                _lib = lib
    return _lib


def lib():
    return load_library()


def status_text(rc: int) -> str:
    return lib().dcg_status_string(rc).decode()


def check(rc: int, info: int = 0, what: str = ""):
    """Map a C status to the reference's exception types (errors.py)."""
    if rc == DCG_OK:
        return
    msg = f"{what}: {status_text(rc)}" if what else status_text(rc)
    if rc == DCG_E_DIMENSION:
        raise DimensionMismatch(msg)
    if rc == DCG_E_NOT_PD:
        raise NotPositiveDefinite(int(info))
    if rc == DCG_E_BREAKDOWN:
        raise BreakdownZeroCurvature(int(info))
    if rc == DCG_E_GRAM_NOT_SPD:
        raise GramNotSpd(f"W'AW not SPD (pivot {int(info)})")
    if rc == DCG_E_BASIS_DEFICIENT:
        raise BasisDeficient(int(info))
    if rc == DCG_E_NO_CONVERGENCE:
        raise NoConvergence(int(info))
    if rc in (DCG_E_ASYMMETRIC,):
        raise ValueError("matrix is not symmetric within tolerance")
    if rc == DCG_E_CONFIG:
        raise ValueError(msg)
    raise DeviceError(msg)


def context(device: int, slot: int = 0) -> int:
    """dcg_context per (device, slot), created lazily and kept for the process.

    Slot 0 serves the caller's current stream; slot 1 the side stream that
    runs the asynchronous Ritz extraction (each context owns its workspace, so
    work in flight on the two streams never shares scratch memory)."""
    key = (device, slot)
    ctx = _contexts.get(key)
    if ctx is None:
        with _lock:
            ctx = _contexts.get(key)
            if ctx is None:
                out = _P()
                check(lib().dcg_context_create(device, ctypes.byref(out)), what="dcg_context_create")
                ctx = out.value
                _contexts[key] = ctx
    return ctx


def grid(device: int) -> tuple[int, int]:
    b, s = ctypes.c_int(), ctypes.c_int()
    check(lib().dcg_context_grid(context(device), ctypes.byref(b), ctypes.byref(s)))
    return b.value, s.value


def launch_count() -> int:
    """Kernels launched by this process through the library so far."""
    return int(lib().dcg_launch_count())
