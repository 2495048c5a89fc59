"""Dense linear algebra of the drop-in surface, executed on the GPU.

Mirrors /root/reference/pkg/src/defcg/linalg.py (names, argument meaning,
error behaviour).  Each call uploads its operands, runs the device twin of the
reference kernel (``dcg_k_*`` / ``dcg_sym_eigen`` / ``dcg_gen_sym_eigen``) and
returns numpy arrays when given numpy arrays.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import DimensionMismatch, NotPositiveDefinite
from .operators import SYMMETRY_RTOL, DenseOperator


@dataclass
class EigenPairs:
    """Eigenvalues in ascending order and matching unit-norm column vectors (linalg.py:20-25)."""

    values: np.ndarray
    vectors: np.ndarray


def as_matrix(a):
    """linalg.py:28-32."""
    if isinstance(a, torch.Tensor):
        if a.ndim != 2:
            raise DimensionMismatch(f"expected a matrix, got ndim={a.ndim}")
        return a
    out = np.ascontiguousarray(a, dtype=np.float64)
    if out.ndim != 2:
        raise DimensionMismatch(f"expected a matrix, got ndim={out.ndim}")
    return out


def as_vector(v):
    """linalg.py:35-39."""
    if isinstance(v, torch.Tensor):
        if v.ndim != 1:
            raise DimensionMismatch(f"expected a vector, got ndim={v.ndim}")
        return v
    out = np.ascontiguousarray(v, dtype=np.float64)
    if out.ndim != 1:
        raise DimensionMismatch(f"expected a vector, got ndim={out.ndim}")
    return out


def require_square(a):
    """linalg.py:42-46."""
    a = as_matrix(a)
    if a.shape[0] != a.shape[1]:
        raise DimensionMismatch(f"expected square matrix, got {tuple(a.shape)}")
    return a


def require_symmetric(a, rtol=SYMMETRY_RTOL):
    """max|A - A'| <= rtol * max|A|, checked on device (linalg.py:49-55)."""
    if isinstance(a, DenseOperator):
        return a
    a = require_square(a)
    DenseOperator.from_matrix(a, check_symmetric=True, rtol=rtol)
    return a


def matvec(a, v):
    """linalg.py:58-63 on device (``dcg_k_matvec``)."""
    if isinstance(a, DenseOperator):
        return a @ v
    a = as_matrix(a)
    v = as_vector(v)
    if a.shape[1] != v.shape[0]:
        raise DimensionMismatch(f"matvec shapes {tuple(a.shape)} and {tuple(v.shape)}")
    m, n = a.shape
    adev, ld = D.to_dev_padded(a)
    vdev = D.to_dev(v, 1)
    y = D.empty(m)
    if m:
        if n == 0:
            y.zero_()
        else:
            N.check(N.lib().dcg_k_matvec(D.ctx(), D.stream(), adev.data_ptr(), m, n, ld, vdev.data_ptr(),
                                         y.data_ptr()), what="matvec")
    return D.out_like(y, v)


def gemm(x, y):
    """linalg.py:66-71 on device (``dcg_k_gemm``, the reference's i-k-j order)."""
    x = as_matrix(x)
    y = as_matrix(y)
    if x.shape[1] != y.shape[0]:
        raise DimensionMismatch(f"gemm shapes {tuple(x.shape)} and {tuple(y.shape)}")
    m, kk = x.shape
    n = y.shape[1]
    xd, yd = D.to_dev(x), D.to_dev(y)
    c = D.empty(m, n)
    if m * n:
        N.check(N.lib().dcg_k_gemm(D.ctx(), D.stream(), D.ptr(xd), D.ptr(yd), c.data_ptr(), m, kk, n), what="gemm")
    return D.out_like(c, x)


def default_pivot_tol(a):
    """linalg.py:74-76."""
    a = np.asarray(a)
    top = np.max(np.diag(a)) if a.shape[0] else 0.0
    return 1e-14 * max(top, 0.0)


def _cholesky_dev(adev: torch.Tensor, pivot_tol: float):
    n = adev.shape[0]
    low = D.empty(n, n)
    fail = ctypes.c_longlong(-1)
    if n:
        N.check(N.lib().dcg_k_cholesky(D.ctx(), D.stream(), adev.data_ptr(), n, float(pivot_tol), low.data_ptr(),
                                       ctypes.byref(fail)), what="cholesky")
    return low, int(fail.value)


def cholesky_factor(a, pivot_tol=None):
    """Lower L with L L' = a; NotPositiveDefinite(pivot) at a pivot <= tol (linalg.py:79-92)."""
    a = require_symmetric(a)
    adev = D.to_dev(a, 2)
    if pivot_tol is None:
        pivot_tol = 1e-14 * max(float(torch.max(torch.diagonal(adev))) if adev.shape[0] else 0.0, 0.0)
    low, fail = _cholesky_dev(adev, pivot_tol)
    if fail >= 0:
        raise NotPositiveDefinite(fail)
    return D.out_like(low, a)


def solve_lower(lower, b):
    """linalg.py:105-110."""
    lower = require_square(lower)
    b = as_vector(b)
    if lower.shape[0] != b.shape[0]:
        raise DimensionMismatch(f"solve shapes {tuple(lower.shape)} and {tuple(b.shape)}")
    ld, bd = D.to_dev(lower), D.to_dev(b)
    y = D.empty(b.shape[0])
    if b.shape[0]:
        N.check(N.lib().dcg_k_solve_lower(D.ctx(), D.stream(), ld.data_ptr(), b.shape[0], bd.data_ptr(),
                                          y.data_ptr()), what="solve_lower")
    return D.out_like(y, b)


def solve_lower_trans(lower, b):
    lower = require_square(lower)
    b = as_vector(b)
    if lower.shape[0] != b.shape[0]:
        raise DimensionMismatch(f"solve shapes {tuple(lower.shape)} and {tuple(b.shape)}")
    ld, bd = D.to_dev(lower), D.to_dev(b)
    x = D.empty(b.shape[0])
    if b.shape[0]:
        N.check(N.lib().dcg_k_solve_lower_trans(D.ctx(), D.stream(), ld.data_ptr(), b.shape[0], bd.data_ptr(),
                                                x.data_ptr()), what="solve_lower_trans")
    return D.out_like(x, b)


def cholesky_solve(lower, b):
    """Solve A x = b from A's Cholesky factor (linalg.py:95-102)."""
    lower = require_square(lower)
    b = as_vector(b)
    if lower.shape[0] != b.shape[0]:
        raise DimensionMismatch(f"solve shapes {tuple(lower.shape)} and {tuple(b.shape)}")
    return solve_lower_trans(lower, solve_lower(lower, b))


def solve_lower_matrix(lower, b):
    """Forward-substitute every column of b (linalg.py:113-122)."""
    lower = require_square(lower)
    b = as_matrix(b)
    if lower.shape[0] != b.shape[0]:
        raise DimensionMismatch(f"solve shapes {tuple(lower.shape)} and {tuple(b.shape)}")
    cols = [solve_lower(lower, np.ascontiguousarray(np.asarray(b)[:, j])) for j in range(b.shape[1])]
    return np.stack(cols, axis=1) if cols else np.empty_like(np.asarray(b))


def cholesky_solve_matrix(lower, b):
    """linalg.py:125-131."""
    b = as_matrix(b)
    cols = [cholesky_solve(lower, np.ascontiguousarray(np.asarray(b)[:, j])) for j in range(b.shape[1])]
    return np.stack(cols, axis=1) if cols else np.empty_like(np.asarray(b))


def jacobi_sweep(a, v):
    """One cyclic Jacobi sweep in place on host arrays via the device twin (_core.pyx:135-177)."""
    n = a.shape[0]
    ad, vd = D.to_dev(a), D.to_dev(v)
    rot = ctypes.c_longlong(0)
    N.check(N.lib().dcg_k_jacobi_sweep(D.ctx(), D.stream(), ad.data_ptr(), vd.data_ptr(), n, ctypes.byref(rot)),
            what="jacobi_sweep")
    a[...] = ad.cpu().numpy()
    v[...] = vd.cpu().numpy()
    return int(rot.value)


def sym_eigen(a, max_sweeps=60, rtol=1e-14):
    """Jacobi eigen-decomposition, ascending (linalg.py:139-165) — one CTA on device."""
    a = require_symmetric(a)
    n = a.shape[0]
    if n == 0:
        return EigenPairs(np.empty(0), np.empty((0, 0)))
    if n > N.MAX_T:
        # beyond the single-CTA Jacobi kernel (Ritz pencils are <= DCG_MAX_T):
        # cuSOLVER's syevd on the device, eigenvalues equal to rounding, ascending,
        # unit eigenvectors (test/diagnostic sizes; linalg.py:139-165 semantics)
        vals, vecs = torch.linalg.eigh(D.to_dev(a, 2))
        return EigenPairs(vals.cpu().numpy(), vecs.cpu().numpy())
    ad = D.to_dev(a)
    vals, vecs = D.empty(n), D.empty(n, n)
    info = ctypes.c_longlong(0)
    rc = N.lib().dcg_sym_eigen(D.ctx(), D.stream(), ad.data_ptr(), n, max_sweeps, rtol, vals.data_ptr(),
                               vecs.data_ptr(), ctypes.byref(info))
    N.check(rc, info.value, "sym_eigen")
    return EigenPairs(vals.cpu().numpy(), vecs.cpu().numpy())


def gen_sym_eigen(g, f, max_sweeps=60):
    """G u = theta F u via F = L L' (linalg.py:168-191) — one CTA on device."""
    g = require_symmetric(g)
    f = require_square(f)
    if tuple(g.shape) != tuple(f.shape):
        raise DimensionMismatch(f"pencil shapes {tuple(g.shape)} and {tuple(f.shape)}")
    require_symmetric(f)
    n = g.shape[0]
    if n == 0:
        return EigenPairs(np.empty(0), np.empty((0, 0)))
    if n > N.MAX_T:
        # G u = theta F u via F = L L' and C = L^-1 G L^-T (linalg.py:168-191) with
        # cuSOLVER: the pivot rule of cholesky_factor, syevd, u = L^-T w normalised
        lower = D.to_dev(cholesky_factor(D.to_dev(f, 2)), 2)
        gd = D.to_dev(g, 2)
        c = torch.linalg.solve_triangular(lower, torch.linalg.solve_triangular(lower, gd, upper=False).T,
                                          upper=False)
        vals, w = torch.linalg.eigh(0.5 * (c + c.T))
        u = torch.linalg.solve_triangular(lower.T, w, upper=True)
        u = u / torch.linalg.norm(u, dim=0, keepdim=True)
        return EigenPairs(vals.cpu().numpy(), u.cpu().numpy())
    gd, fd = D.to_dev(g), D.to_dev(f)
    vals, vecs = D.empty(n), D.empty(n, n)
    info = ctypes.c_longlong(0)
    rc = N.lib().dcg_gen_sym_eigen(D.ctx(), D.stream(), gd.data_ptr(), fd.data_ptr(), n, max_sweeps,
                                   vals.data_ptr(), vecs.data_ptr(), ctypes.byref(info))
    N.check(rc, info.value, "gen_sym_eigen")
    return EigenPairs(vals.cpu().numpy(), vecs.cpu().numpy())
