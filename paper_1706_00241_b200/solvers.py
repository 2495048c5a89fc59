"""Conjugate gradients and deflated CG — the drop-in for defcg.solvers.

Same public names, signatures, defaults and return types as
/root/reference/pkg/src/defcg/solvers.py (``SolverConfig``, ``KrylovLog``,
``SolveReport``, ``RecycleBasis``, ``empty_basis``, ``cg_solve``,
``deflated_cg_solve``, ``apply_deflation_projector``).  The iteration itself
(``_run_loop``, solvers.py:131-204, plus the warm-start correction of
deflated_cg_solve, solvers.py:222-239) runs as ONE persistent cooperative
CUDA kernel (``dcg_solve``): the matrix never leaves HBM, the residual
history and the Krylov log are written on device, and the host synchronises
once per solve.  An empty basis takes the plain-CG path of the same kernel,
so k = 0 def-CG is bit-identical to CG exactly as in the reference.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import DimensionMismatch, GramNotSpd
from .operators import DenseOperator, as_operator

TERM_CONVERGED = "converged"
TERM_MAX_ITERS = "max_iters"


@dataclass(frozen=True)
class SolverConfig:
    """Stopping rule and logging window (solvers.py:28-51)."""

    tol: float = 1e-5
    max_iters: int | None = None
    ell: int = 12
    recompute_residual_every: int = 50

    def __post_init__(self):
        if self.tol <= 0.0:
            raise ValueError("tol must be positive")
        if self.ell < 0:
            raise ValueError("ell must be non-negative")
        if self.max_iters is not None and self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if self.recompute_residual_every < 0:
            raise ValueError("recompute_residual_every must be non-negative")

    def c_struct(self) -> N.CSolverConfig:
        c = N.CSolverConfig()
        c.tol = self.tol
        c.max_iters = 0 if self.max_iters is None else int(self.max_iters)
        c.ell = int(self.ell)
        c.recompute_residual_every = int(self.recompute_residual_every)
        return c


class KrylovLog:
    """Per-iteration quantities of the first min(ell, iterations) steps
    (solvers.py:54-72), resident on device.  ``p``, ``r``, ``d``, ``alpha``,
    ``beta`` and ``mu`` materialise as lists of numpy arrays / floats on first
    access; ``p_dev``/``r_dev``/``alpha_dev`` are the device views the
    extraction kernel consumes."""

    def __init__(self, n: int, ell: int, k: int):
        self.n = n
        self.capacity = ell
        self.k = k
        self.m = 0
        cap = max(ell, 0)
        self._p = D.empty(max(cap, 1), max(n, 1))
        self._r = D.empty(cap + 1, max(n, 1))
        self._s = D.empty(3, max(cap, 1))   # d, alpha, beta
        self._mu = D.empty(max(cap, 1), max(k, 1))
        self._host = None

    def c_struct(self) -> N.CKrylovLog:
        c = N.CKrylovLog()
        c.ell = self.capacity
        c.d_p = self._p.data_ptr()
        c.d_r = self._r.data_ptr()
        c.d_d = self._s[0].data_ptr()
        c.d_alpha = self._s[1].data_ptr()
        c.d_beta = self._s[2].data_ptr()
        c.d_mu = self._mu.data_ptr()
        return c

    @property
    def stored_iterations(self):
        return self.m

    @property
    def p_dev(self):
        return self._p[: self.m, : self.n]

    @property
    def r_dev(self):
        return self._r[: self.m + 1, : self.n]

    @property
    def alpha_dev(self):
        return self._s[1, : self.m]

    def _materialise(self):
        if self._host is None:
            m, n = self.m, self.n
            s = self._s[:, :m].cpu().numpy()
            self._host = {
                "p": [row.copy() for row in self._p[:m, :n].cpu().numpy()],
                "r": [row.copy() for row in self._r[: m + 1, :n].cpu().numpy()],
                "d": [float(v) for v in s[0]],
                "alpha": [float(v) for v in s[1]],
                "beta": [float(v) for v in s[2]],
                "mu": [row.copy() for row in self._mu[:m, : self.k].cpu().numpy()] if self.k else [],
            }
        return self._host

    p = property(lambda self: self._materialise()["p"])
    r = property(lambda self: self._materialise()["r"])
    d = property(lambda self: self._materialise()["d"])
    alpha = property(lambda self: self._materialise()["alpha"])
    beta = property(lambda self: self._materialise()["beta"])
    mu = property(lambda self: self._materialise()["mu"])


@dataclass
class SolveReport:
    """solvers.py:75-81, plus the solve kernel's device time."""

    iterations: int
    residual_history: list
    converged: bool
    wall_time: float
    termination: str
    device_ms: float = 0.0


class RecycleBasis:
    """Deflation space W with its image AW and the cached Cholesky factor of
    W'AW (solvers.py:84-115).  Columns live on device as row-major n x k
    blocks; ``w``/``aw``/``gram_chol`` are numpy views materialised on access."""

    def __init__(self, w, aw, gram_chol=None):
        if not isinstance(w, torch.Tensor):
            w = np.ascontiguousarray(w, dtype=np.float64)
        if not isinstance(aw, torch.Tensor):
            aw = np.ascontiguousarray(aw, dtype=np.float64)
        if w.ndim != 2 or aw.ndim != 2:
            raise DimensionMismatch(f"expected a matrix, got ndim={w.ndim}/{aw.ndim}")
        if tuple(w.shape) != tuple(aw.shape):
            raise DimensionMismatch(f"W {tuple(w.shape)} and AW {tuple(aw.shape)} differ")
        self.w_dev = D.to_dev(w, 2)
        self.aw_dev = D.to_dev(aw, 2)
        self.chol_dev = None if gram_chol is None else D.to_dev(gram_chol, 2)

    @property
    def k(self):
        return self.w_dev.shape[1]

    @property
    def n(self):
        return self.w_dev.shape[0]

    @property
    def w(self):
        return self.w_dev.cpu().numpy()

    @property
    def aw(self):
        return self.aw_dev.cpu().numpy()

    @property
    def gram_chol(self):
        return None if self.chol_dev is None else self.chol_dev.cpu().numpy()

    @gram_chol.setter
    def gram_chol(self, value):
        self.chol_dev = None if value is None else D.to_dev(value, 2)

    def ensure_factored_dev(self) -> torch.Tensor:
        """Cholesky of sym(W'AW) on device; GramNotSpd on failure (solvers.py:107-115)."""
        if self.chol_dev is None:
            k = self.k
            chol = D.empty(max(k, 1), max(k, 1))
            if k:
                kout, info = ctypes.c_longlong(k), ctypes.c_longlong(0)
                rc = N.lib().dcg_gram_factor(D.ctx(), D.stream(), self.w_dev.data_ptr(), self.aw_dev.data_ptr(),
                                             self.n, k, 0, chol.data_ptr(), ctypes.byref(kout), ctypes.byref(info))
                if rc == N.DCG_E_GRAM_NOT_SPD:
                    raise GramNotSpd(f"W'AW not SPD (pivot {info.value})")
                N.check(rc, info.value, "gram_factor")
            self.chol_dev = chol[:k, :k]
        return self.chol_dev

    def ensure_factored(self):
        self.ensure_factored_dev()
        return self.gram_chol

    def c_struct(self) -> N.CBasis:
        b = N.CBasis()
        b.k = self.k
        b.d_w = self.w_dev.data_ptr() if self.k else None
        b.d_aw = self.aw_dev.data_ptr() if self.k else None
        b.d_chol = self.chol_dev.contiguous().data_ptr() if (self.k and self.chol_dev is not None) else None
        return b


def empty_basis(n):
    """solvers.py:118-119."""
    return RecycleBasis(np.empty((n, 0)), np.empty((n, 0)), np.empty((0, 0)))


# ---------------------------------------------------------------------------
# device solve
# ---------------------------------------------------------------------------


def _solve_dev(op: DenseOperator, b: torch.Tensor, x0: torch.Tensor, basis: RecycleBasis | None,
               cfg: SolverConfig, t_start: float):
    """One call of the persistent solve kernel.  Returns (x, report, log) with
    x on device."""
    n = op.n
    k = basis.k if basis is not None else 0
    if k:
        basis.ensure_factored_dev()
        if basis.chol_dev is not None and not basis.chol_dev.is_contiguous():
            basis.chol_dev = basis.chol_dev.contiguous()
    log = KrylovLog(n, cfg.ell, k)
    max_iters = 10 * n if cfg.max_iters is None else cfg.max_iters
    hist = D.empty(max_iters + 1)
    x = D.empty(max(n, 1))
    if n == 0:
        log.m = 0
        rep = SolveReport(0, [0.0], True, time.perf_counter() - t_start, TERM_CONVERGED)
        return x[:0], rep, log
    cop = op.c_struct()
    cb = basis.c_struct() if k else None
    ccfg = cfg.c_struct()
    clog = log.c_struct()
    info = N.CSolveInfo()
    err = ctypes.c_longlong(0)
    rc = N.lib().dcg_solve(D.ctx(), D.stream(), ctypes.byref(cop), b.data_ptr(), x0.data_ptr(),
                           ctypes.byref(cb) if cb is not None else None, ctypes.byref(ccfg), x.data_ptr(),
                           ctypes.byref(clog), hist.data_ptr(), ctypes.byref(info), ctypes.byref(err))
    N.check(rc, err.value, "solve")
    its = int(info.iterations)
    log.m = int(info.stored)
    history = hist[: its + 1].cpu().tolist()
    conv = bool(info.converged)
    rep = SolveReport(its, history, conv, time.perf_counter() - t_start, TERM_CONVERGED if conv else TERM_MAX_ITERS,
                      float(info.device_ms))
    return x[:n], rep, log


def _check_system(a, b, x0):
    """solvers.py:122-128: operator, b, x0 validated and placed on device."""
    op = as_operator(a)
    bd = D.to_dev(b, 1)
    xd = D.to_dev(x0, 1)
    if op.n != bd.shape[0] or bd.shape[0] != xd.shape[0]:
        raise DimensionMismatch(f"system shapes {op.shape}, {tuple(bd.shape)}, {tuple(xd.shape)}")
    return op, bd, xd


def cg_solve(a, b, x0=None, cfg=None):
    """Standard CG with relative-residual stopping (solvers.py:207-219).

    Returns (x, SolveReport, KrylovLog); the log's mu list is empty."""
    cfg = cfg or SolverConfig()
    if not isinstance(b, torch.Tensor):
        b = D.as_host_vector(b)
    elif b.ndim != 1:
        raise DimensionMismatch(f"expected a vector, got ndim={b.ndim}")
    if x0 is None:
        x0 = torch.zeros_like(b, dtype=D.F64) if isinstance(b, torch.Tensor) else np.zeros(b.shape[0])
    t0 = time.perf_counter()
    op, bd, xd = _check_system(a, b, x0)
    x, rep, log = _solve_dev(op, bd, xd, None, cfg, t0)
    return D.out_like(x, b), rep, log


def deflated_cg_solve(a, b, x_prev, basis, cfg=None):
    """Deflated CG over span(basis.w), warm-started from x_prev corrected
    into W'r = 0 (solvers.py:222-239).  An empty basis is exactly cg_solve."""
    cfg = cfg or SolverConfig()
    t0 = time.perf_counter()
    op, bd, xd = _check_system(a, b, x_prev)
    if basis.k == 0:
        x, rep, log = _solve_dev(op, bd, xd, None, cfg, t0)
        return D.out_like(x, b), rep, log
    if basis.n != bd.shape[0]:
        raise DimensionMismatch(f"basis rows {basis.n} vs system size {bd.shape[0]}")
    x, rep, log = _solve_dev(op, bd, xd, basis, cfg, t0)
    return D.out_like(x, b), rep, log


def apply_deflation_projector(a, basis, v):
    """P_W v = v - AW (W'AW)^-1 W' v (solvers.py:242-256); ``basis`` must carry
    AW for this ``a``."""
    if isinstance(a, DenseOperator):
        shape = a.shape
    else:
        if not isinstance(a, torch.Tensor):
            a = np.ascontiguousarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise DimensionMismatch(f"expected a matrix, got ndim={a.ndim}")
        shape = tuple(a.shape)
    if not isinstance(v, torch.Tensor):
        v = D.as_host_vector(v)
    if shape[1] != v.shape[0]:
        raise DimensionMismatch(f"matrix {shape} vs vector size {v.shape[0]}")
    if basis.k == 0:
        return v.clone() if isinstance(v, torch.Tensor) else v.copy()
    if basis.n != v.shape[0]:
        raise DimensionMismatch(f"basis rows {basis.n} vs vector size {v.shape[0]}")
    basis.ensure_factored_dev()
    vd = D.to_dev(v, 1)
    out = D.empty(vd.shape[0])
    cb = basis.c_struct()
    N.check(N.lib().dcg_deflation_project(D.ctx(), D.stream(), vd.shape[0], ctypes.byref(cb), vd.data_ptr(),
                                          out.data_ptr()), what="deflation_project")
    return D.out_like(out, v)
