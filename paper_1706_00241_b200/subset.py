"""Random subset-of-data baseline for the cost/accuracy comparison, on device
(reference: /root/reference/pkg/src/defcg/subset.py:38-98).

Fits the Laplace mode on a seeded uniform random subset of m points with the
direct (Cholesky) solver -- K_mm assembled on device, cuSOLVER's potrf with the
reference's pivot-tolerance semantics (gpc._dense_cholesky_factor) -- then
induces the other latents from the conditional mean K_(n-m)m K_mm^-1 f_m
(the cross block from ``dcg_k_rbf_cross``, the product on the row GEMV) and
scores the whole training set with them.  The subset indices come from the
same ``numpy.random.default_rng(seed).choice`` call as the reference's, so a
seed selects the same points.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from .errors import ConfigError
from .gpc import (
    SOLVER_CHOLESKY,
    _dense_cholesky_factor,
    laplace_newton,
    likelihood_derivs,
    rbf_cross_kernel,
    rbf_kernel,
)
from .linalg import matvec
from .operators import DenseOperator


class SubsetModel:
    """Fitted subset: chosen indices, kernel blocks and subset latents
    (subset.py:20-35).  Blocks built by ``fit_subset`` stay on the device
    (``*_dev``); the numpy fields materialise on first access.  A model built
    from numpy arrays (as the reference's tests do) is moved to the device
    when used."""

    def __init__(self, indices_m, rest_indices, k_mm, k_rest_m, f_m):
        self.indices_m = np.asarray(indices_m)
        self.rest_indices = np.asarray(rest_indices)
        self._k_mm, self._k_rest_m, self._f_m = k_mm, k_rest_m, f_m

    @staticmethod
    def _host(v):
        if isinstance(v, DenseOperator):
            return np.asarray(v)
        if isinstance(v, torch.Tensor):
            return v.detach().cpu().numpy()
        return v

    @property
    def k_mm(self):
        self._k_mm = self._host(self._k_mm)
        return self._k_mm

    @property
    def k_rest_m(self):
        self._k_rest_m = self._host(self._k_rest_m)
        return self._k_rest_m

    @property
    def f_m(self):
        self._f_m = self._host(self._f_m)
        return self._f_m

    @property
    def m(self):
        return self.indices_m.shape[0]

    @property
    def n(self):
        return self.indices_m.shape[0] + self.rest_indices.shape[0]


def fit_subset(x, y, fraction, params, newton_tol=1.0, seed=0, jitter=None, max_newton=30):
    """Fit the Laplace mode on a seeded uniform random subset (subset.py:38-68).

    Returns (SubsetModel, Newton records of the subset fit)."""
    xh = x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x, dtype=np.float64)
    if xh.ndim != 2:
        raise ConfigError(f"expected a data matrix, got ndim={xh.ndim}")
    yh = y.detach().cpu().numpy() if isinstance(y, torch.Tensor) else np.asarray(y)
    n = xh.shape[0]
    if not 0.0 < fraction <= 1.0:
        raise ConfigError(f"fraction must be in (0, 1], got {fraction}")
    if fraction * n < 1.0:
        raise ConfigError(f"fraction {fraction} selects no points from n={n}")
    m = min(n, max(1, int(round(fraction * n))))
    rng = np.random.default_rng(seed)
    indices = rng.choice(n, size=m, replace=False)
    rest = np.setdiff1d(np.arange(n), indices)
    xd = D.to_dev(xh, 2)
    idx_d = torch.from_numpy(indices).to(xd.device)
    k_mm = rbf_kernel(xd.index_select(0, idx_d), params, jitter)
    state, records = laplace_newton(k_mm, yh[indices], solver=SOLVER_CHOLESKY, newton_tol=newton_tol,
                                    max_newton=max_newton)
    if rest.size:
        k_rest_m = rbf_cross_kernel(xd.index_select(0, torch.from_numpy(rest).to(xd.device)),
                                    xd.index_select(0, idx_d), params)
    else:
        k_rest_m = D.empty(0, m)
    return SubsetModel(indices, rest, k_mm, k_rest_m, state.f), records


def _induce_dev(model, f_m=None) -> torch.Tensor:
    f = D.to_dev(model._f_m if f_m is None else f_m, 1)
    if model.rest_indices.size == 0:
        return D.empty(0)
    k_mm = model._k_mm if isinstance(model._k_mm, DenseOperator) else DenseOperator.from_matrix(model._k_mm)
    lower = _dense_cholesky_factor(k_mm.kernel_view())                     # cholesky_factor, linalg.py:79-92
    alpha = torch.cholesky_solve(f[:, None], lower)[:, 0]                  # cholesky_solve, linalg.py:95-102
    return matvec(D.to_dev(model._k_rest_m, 2), alpha)                     # linalg.py:58-63 (device GEMV)


def induce_latents(model, f_m=None):
    """Conditional-mean latents for the points outside the subset (subset.py:71-77)."""
    out = _induce_dev(model, f_m)
    return out if isinstance(f_m, torch.Tensor) else out.cpu().numpy()


def assemble_full_latents(model, f_m=None):
    """Full-length latent vector in original data order (subset.py:80-87)."""
    fm = D.to_dev(model._f_m if f_m is None else f_m, 1)
    f = D.empty(model.n)
    dev = f.device
    f[torch.from_numpy(model.indices_m).to(dev)] = fm
    if model.rest_indices.size:
        f[torch.from_numpy(model.rest_indices).to(dev)] = _induce_dev(model, fm)
    return f if isinstance(f_m, torch.Tensor) else f.cpu().numpy()


def evaluate_full(model, x, y):
    """log p(y|f) over all n points with subset + induced latents (subset.py:90-98)."""
    nx, ny = int(np.shape(x)[0]) if not isinstance(x, torch.Tensor) else int(x.shape[0]), len(y)
    if nx != ny or ny != model.n:
        raise ConfigError("data size does not match the fitted model")
    f = assemble_full_latents(model)
    loglik, _, _ = likelihood_derivs(f, y)
    return loglik
