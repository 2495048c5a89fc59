"""Device twin of the reference's kernel-backend plugin (``defcg._kernels``).

The reference selects a module exporting ``NAME, matvec, gemm, cholesky,
solve_lower, solve_lower_trans, rbf_gram, rbf_cross, jacobi_sweep`` through
``DEFCG_BACKEND`` (/root/reference/pkg/src/defcg/_kernels/__init__.py:11-45).
This module exports the same nine names with the same signatures and return
conventions (``cholesky`` -> ``(L, fail_index)``, ``jacobi_sweep`` mutates its
arguments and returns the rotation count), each running the ``dcg_k_*`` CUDA
kernel.  It serves unit parity against ``_core.pyx``; the solvers use the
fused device path instead of per-call host round trips.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device as D
from . import _native as N
from . import linalg as _linalg

NAME = "cuda-sm100a"


def matvec(a, x):
    """_core.pyx:16-28."""
    return _linalg.matvec(a, x)


def gemm(a, b):
    """_core.pyx:31-44 (i-k-j order, bit-identical)."""
    return _linalg.gemm(a, b)


def cholesky(a, pivot_tol):
    """_core.pyx:47-66: returns (L, j) with j the first failing pivot or -1."""
    ad = D.to_dev(a, 2)
    low, fail = _linalg._cholesky_dev(ad, float(pivot_tol))
    return D.out_like(low, a), fail


def solve_lower(lower, b):
    """_core.pyx:69-80."""
    return _linalg.solve_lower(lower, b)


def solve_lower_trans(lower, b):
    """_core.pyx:83-94."""
    return _linalg.solve_lower_trans(lower, b)


def rbf_gram(x, signal_var, inv_two_ell2, jitter):
    """_core.pyx:97-114: exact symmetry, exact diagonal signal_var + jitter."""
    xd = D.to_dev(x, 2)
    n, dim = xd.shape
    out = D.empty(n, n)
    if n:
        N.check(N.lib().dcg_k_rbf_gram(D.ctx(), D.stream(), xd.data_ptr(), n, dim, float(signal_var),
                                       float(inv_two_ell2), float(jitter), out.data_ptr(), n, 0, n), what="rbf_gram")
    return D.out_like(out, x)


def rbf_cross(xa, xb, signal_var, inv_two_ell2):
    """_core.pyx:117-132."""
    ad, bd = D.to_dev(xa, 2), D.to_dev(xb, 2)
    out = D.empty(ad.shape[0], bd.shape[0])
    if out.numel():
        N.check(N.lib().dcg_k_rbf_cross(D.ctx(), D.stream(), ad.data_ptr(), ad.shape[0], bd.data_ptr(), bd.shape[0],
                                        ad.shape[1], float(signal_var), float(inv_two_ell2), out.data_ptr()),
                what="rbf_cross")
    return D.out_like(out, xa)


def jacobi_sweep(a, v):
    """_core.pyx:135-177: one cyclic sweep in place; returns the rotation count."""
    return _linalg.jacobi_sweep(a, v)
