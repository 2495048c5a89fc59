"""CPU oracle for the def-CG hot path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it; the
product package (``paper_1706_00241_b200``) never does, and fails loudly when
its CUDA library is missing instead of falling back here.

It restates, function for function, the reference package ``defcg`` (arXiv
1706.00241) along the solve-sequence path named by BASELINE.json's north_star:

* kernel backends (``_kernels``): the compiled core is restated in C
  (``oracle/core.c``, bit-identical to ``_core.pyx``) and the numpy fallback
  in numpy (``_kernels/_ref.py``); ``backend=`` selects one, exactly like
  ``DEFCG_BACKEND`` (``_kernels/__init__.py:11-23``);
* ``linalg.py`` (validation, Cholesky with pivot tolerance, cyclic Jacobi,
  generalised eigenproblem), ``solvers.py`` (the shared CG / def-CG loop),
  ``recycle.py`` (refresh, harmonic-Ritz extraction, ``solve_next``) and the
  ``gpc.py`` Laplace-Newton driver, each citing the lines it follows.

Parity is pinned: ``tests/test_oracle.py`` checks this module against golden
vectors produced by running the reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liboracle_core.so"

# --------------------------------------------------------------------------
# errors (reference errors.py:8-93) — oracle-local classes, same payloads
# --------------------------------------------------------------------------


class OracleError(Exception):
    pass


class ONotPositiveDefinite(OracleError):
    def __init__(self, pivot_index):
        self.pivot_index = pivot_index
        super().__init__(f"non-positive pivot at index {pivot_index}")


class ONoConvergence(OracleError):
    def __init__(self, sweeps):
        self.sweeps = sweeps
        super().__init__(f"no convergence after {sweeps} sweeps")


class OBreakdown(OracleError):
    def __init__(self, iteration):
        self.iteration = iteration
        super().__init__(f"non-positive curvature at iteration {iteration}")


class OGramNotSpd(OracleError):
    pass


class OBasisDeficient(OracleError):
    def __init__(self, remaining):
        self.remaining = remaining
        super().__init__(f"only {remaining} independent basis columns remain")


class OStateInconsistent(OracleError):
    pass


class ONoProgress(OracleError):
    pass


class ODimensionMismatch(OracleError):
    pass


# --------------------------------------------------------------------------
# kernel backends
# --------------------------------------------------------------------------


def build_core(force: bool = False) -> Path:
    """Compile core.c (gcc, -O3, no FMA contraction) into oracle/_build."""
    src = HERE / "core.c"
    if not force and LIB_PATH.exists() and LIB_PATH.stat().st_mtime >= src.stat().st_mtime:
        return LIB_PATH
    LIB_PATH.parent.mkdir(exist_ok=True)
    cc = os.environ.get("CC", "gcc")
    cmd = [cc, "-O3", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math", "-o", str(LIB_PATH), str(src), "-lm"]
    subprocess.run(cmd, check=True, capture_output=True)
    return LIB_PATH


_DP = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_longlong


class _CompiledCore:
    """ctypes view of core.c — the restated ``_core`` backend."""

    NAME = "compiled"

    def __init__(self):
        lib = ctypes.CDLL(str(build_core()))
        for name, res, args in [
            ("or_matvec", None, [_DP, _I64, _I64, _DP, _DP]),
            ("or_gemm", None, [_DP, _DP, _DP, _I64, _I64, _I64]),
            ("or_cholesky", _I64, [_DP, _I64, ctypes.c_double, _DP]),
            ("or_solve_lower", None, [_DP, _I64, _DP, _DP]),
            ("or_solve_lower_trans", None, [_DP, _I64, _DP, _DP]),
            ("or_rbf_gram", None, [_DP, _I64, _I64, ctypes.c_double, ctypes.c_double, ctypes.c_double, _DP]),
            ("or_rbf_cross", None, [_DP, _I64, _DP, _I64, _I64, ctypes.c_double, ctypes.c_double, _DP]),
            ("or_jacobi_sweep", _I64, [_DP, _DP, _I64]),
        ]:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        self._lib = lib

    @staticmethod
    def _p(a):
        return a.ctypes.data_as(_DP)

    def matvec(self, a, x):
        a = np.ascontiguousarray(a, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(a.shape[0])
        self._lib.or_matvec(self._p(a), a.shape[0], a.shape[1], self._p(x), self._p(y))
        return y

    def gemm(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        c = np.empty((a.shape[0], b.shape[1]))
        self._lib.or_gemm(self._p(a), self._p(b), self._p(c), a.shape[0], a.shape[1], b.shape[1])
        return c

    def cholesky(self, a, pivot_tol):
        a = np.ascontiguousarray(a, dtype=np.float64)
        out = np.empty_like(a)
        fail = self._lib.or_cholesky(self._p(a), a.shape[0], float(pivot_tol), self._p(out))
        return out, int(fail)

    def solve_lower(self, lower, b):
        lower = np.ascontiguousarray(lower, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        y = np.empty(lower.shape[0])
        self._lib.or_solve_lower(self._p(lower), lower.shape[0], self._p(b), self._p(y))
        return y

    def solve_lower_trans(self, lower, b):
        lower = np.ascontiguousarray(lower, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(lower.shape[0])
        self._lib.or_solve_lower_trans(self._p(lower), lower.shape[0], self._p(b), self._p(x))
        return x

    def rbf_gram(self, x, var, inv2, jitter):
        x = np.ascontiguousarray(x, dtype=np.float64)
        k = np.empty((x.shape[0], x.shape[0]))
        self._lib.or_rbf_gram(self._p(x), x.shape[0], x.shape[1], var, inv2, jitter, self._p(k))
        return k

    def rbf_cross(self, xa, xb, var, inv2):
        xa = np.ascontiguousarray(xa, dtype=np.float64)
        xb = np.ascontiguousarray(xb, dtype=np.float64)
        k = np.empty((xa.shape[0], xb.shape[0]))
        self._lib.or_rbf_cross(self._p(xa), xa.shape[0], self._p(xb), xb.shape[0], xa.shape[1], var, inv2, self._p(k))
        return k

    def jacobi_sweep(self, a, v):
        assert a.flags.c_contiguous and v.flags.c_contiguous
        return int(self._lib.or_jacobi_sweep(self._p(a), self._p(v), a.shape[0]))


class _NumpyCore:
    """Restatement of the numpy fallback backend (``_kernels/_ref.py:15-118``)."""

    NAME = "numpy"

    matvec = staticmethod(lambda a, x: a @ x)
    gemm = staticmethod(lambda a, b: a @ b)

    @staticmethod
    def cholesky(a, pivot_tol):  # _ref.py:23-38
        n = a.shape[0]
        low = np.zeros_like(a)
        for j in range(n):
            piv = a[j, j] - low[j, :j] @ low[j, :j]
            if piv <= pivot_tol:
                return low, j
            root = math.sqrt(piv)
            low[j, j] = root
            if j + 1 < n:
                low[j + 1 :, j] = (a[j + 1 :, j] - low[j + 1 :, :j] @ low[j, :j]) / root
        return low, -1

    @staticmethod
    def solve_lower(lower, b):  # _ref.py:41-46
        out = np.empty_like(b)
        for i in range(lower.shape[0]):
            out[i] = (b[i] - lower[i, :i] @ out[:i]) / lower[i, i]
        return out

    @staticmethod
    def solve_lower_trans(lower, b):  # _ref.py:49-54
        out = np.empty_like(b)
        for i in range(lower.shape[0] - 1, -1, -1):
            out[i] = (b[i] - lower[i + 1 :, i] @ out[i + 1 :]) / lower[i, i]
        return out

    @staticmethod
    def rbf_gram(x, var, inv2, jitter):  # _ref.py:57-66
        sq = np.einsum("ij,ij->i", x, x)
        d2 = sq[:, None] + sq[None, :] - 2.0 * (x @ x.T)
        np.maximum(d2, 0.0, out=d2)
        k = np.tril(var * np.exp(-d2 * inv2), -1)
        k = k + k.T
        np.fill_diagonal(k, var + jitter)
        return k

    @staticmethod
    def rbf_cross(xa, xb, var, inv2):  # _ref.py:69-74
        sqa = np.einsum("ij,ij->i", xa, xa)
        sqb = np.einsum("ij,ij->i", xb, xb)
        d2 = sqa[:, None] + sqb[None, :] - 2.0 * (xa @ xb.T)
        np.maximum(d2, 0.0, out=d2)
        return var * np.exp(-d2 * inv2)

    @staticmethod
    def jacobi_sweep(a, v):  # _ref.py:77-118
        n = a.shape[0]
        count = 0
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = a[p, q]
                g = 100.0 * abs(apq)
                if abs(a[p, p]) + g == abs(a[p, p]) and abs(a[q, q]) + g == abs(a[q, q]):
                    a[p, q] = a[q, p] = 0.0
                    continue
                if apq == 0.0:
                    continue
                tau = (a[q, q] - a[p, p]) / (2.0 * apq)
                t = 1.0 / (tau + math.sqrt(1.0 + tau * tau)) if tau >= 0.0 else -1.0 / (-tau + math.sqrt(1.0 + tau * tau))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = t * c
                cp, cq = a[:, p].copy(), a[:, q].copy()
                a[:, p], a[:, q] = c * cp - s * cq, s * cp + c * cq
                rp, rq = a[p, :].copy(), a[q, :].copy()
                a[p, :], a[q, :] = c * rp - s * rq, s * rp + c * rq
                a[p, q] = a[q, p] = 0.0
                vp, vq = v[:, p].copy(), v[:, q].copy()
                v[:, p], v[:, q] = c * vp - s * vq, s * vp + c * vq
                count += 1
        return count


_BACKENDS: dict = {}


def backend(name: str = "compiled"):
    if name in ("compiled", "cy", "c"):
        key = "compiled"
    elif name in ("numpy", "py", "ref"):
        key = "numpy"
    else:
        raise ValueError(f"unknown backend {name!r}")
    if key not in _BACKENDS:
        _BACKENDS[key] = _CompiledCore() if key == "compiled" else _NumpyCore()
    return _BACKENDS[key]


# --------------------------------------------------------------------------
# dense linear algebra (linalg.py)
# --------------------------------------------------------------------------


def _mat(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ODimensionMismatch(f"expected a matrix, got ndim={a.ndim}")
    return a


def _vec(v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.ndim != 1:
        raise ODimensionMismatch(f"expected a vector, got ndim={v.ndim}")
    return v


def check_symmetric(a, rtol=1e-12):
    """linalg.py:42-55 (square, then max|A-A'| <= rtol max|A|)."""
    a = _mat(a)
    if a.shape[0] != a.shape[1]:
        raise ODimensionMismatch(f"expected square matrix, got {a.shape}")
    if a.size:
        scale = np.max(np.abs(a))
        if np.max(np.abs(a - a.T)) > rtol * max(scale, 1e-300):
            raise ValueError("matrix is not symmetric within tolerance")
    return a


def chol_factor(a, pivot_tol=None, be="compiled"):
    """linalg.py:74-92."""
    a = check_symmetric(a)
    if pivot_tol is None:
        top = np.max(np.diag(a)) if a.shape[0] else 0.0
        pivot_tol = 1e-14 * max(top, 0.0)
    low, fail = backend(be).cholesky(a, float(pivot_tol))
    if fail >= 0:
        raise ONotPositiveDefinite(fail)
    return low


def chol_solve(low, b, be="compiled"):
    """linalg.py:95-102."""
    k = backend(be)
    return k.solve_lower_trans(low, k.solve_lower(low, _vec(b)))


def _lower_solve_cols(low, rhs, be):
    """linalg.py:113-122 (column by column)."""
    out = np.empty_like(rhs)
    for j in range(rhs.shape[1]):
        out[:, j] = backend(be).solve_lower(low, np.ascontiguousarray(rhs[:, j]))
    return out


def sym_eigen(a, max_sweeps=60, rtol=1e-14, be="compiled"):
    """Cyclic Jacobi, ascending stable order (linalg.py:134-165)."""
    a = check_symmetric(a)
    n = a.shape[0]
    if n == 0:
        return np.empty(0), np.empty((0, 0))
    work = a.copy()
    vecs = np.eye(n)
    frob = float(np.sqrt(np.sum(a * a)))
    if frob == 0.0:
        return np.zeros(n), vecs

    def off(m):
        o = m - np.diag(np.diag(m))
        return float(np.sqrt(np.sum(o * o)))

    done = off(work) <= rtol * frob
    for _ in range(max_sweeps):
        if done:
            break
        backend(be).jacobi_sweep(work, vecs)
        done = off(work) <= rtol * frob
    if not done:
        raise ONoConvergence(max_sweeps)
    vals = np.diag(work).copy()
    order = np.argsort(vals, kind="stable")
    return vals[order], np.ascontiguousarray(vecs[:, order])


def gen_sym_eigen(g, f, max_sweeps=60, be="compiled"):
    """G u = theta F u through F = L L' (linalg.py:168-191)."""
    g = check_symmetric(g)
    f = _mat(f)
    if g.shape != f.shape:
        raise ODimensionMismatch(f"pencil shapes {g.shape} and {f.shape}")
    low = chol_factor(f, be=be)
    y = _lower_solve_cols(low, g, be)
    c = _lower_solve_cols(low, np.ascontiguousarray(y.T), be)
    c = 0.5 * (c + c.T)
    vals, w = sym_eigen(c, max_sweeps=max_sweeps, be=be)
    n = g.shape[0]
    vecs = np.empty((n, n))
    for j in range(n):
        u = backend(be).solve_lower_trans(low, np.ascontiguousarray(w[:, j]))
        nrm = float(np.linalg.norm(u))
        vecs[:, j] = u / nrm if nrm > 0.0 else u
    return vals, vecs


# --------------------------------------------------------------------------
# Krylov solvers (solvers.py)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class Cfg:
    """SolverConfig (solvers.py:28-51)."""

    tol: float = 1e-5
    max_iters: int | None = None
    ell: int = 12
    recompute_residual_every: int = 50


@dataclass
class Log:
    """KrylovLog (solvers.py:54-72)."""

    d: list = field(default_factory=list)
    alpha: list = field(default_factory=list)
    beta: list = field(default_factory=list)
    mu: list = field(default_factory=list)
    p: list = field(default_factory=list)
    r: list = field(default_factory=list)


@dataclass
class Report:
    """SolveReport (solvers.py:75-81)."""

    iterations: int
    residual_history: list
    converged: bool
    wall_time: float
    termination: str


@dataclass
class Basis:
    """RecycleBasis (solvers.py:84-115); chol is W'AW's lower factor."""

    w: np.ndarray
    aw: np.ndarray
    chol: np.ndarray | None = None

    @property
    def k(self):
        return self.w.shape[1]

    def factored(self, be="compiled"):
        if self.chol is None:
            gram = self.w.T @ self.aw
            gram = 0.5 * (gram + gram.T)
            try:
                self.chol = chol_factor(gram, be=be)
            except ONotPositiveDefinite as exc:
                raise OGramNotSpd(f"W'AW not SPD (pivot {exc.pivot_index})") from exc
        return self.chol


def _system(a, b, x0):
    """solvers.py:122-128."""
    a = check_symmetric(a)
    b, x0 = _vec(b), _vec(x0)
    if not (a.shape[0] == b.shape[0] == x0.shape[0]):
        raise ODimensionMismatch(f"system shapes {a.shape}, {b.shape}, {x0.shape}")
    return a, b, x0


def krylov_loop(a, b, x0, basis, cfg, t_start, be="compiled"):
    """The shared CG / def-CG iteration, solvers.py:131-204 (basis None = CG)."""
    kern = backend(be)
    n = b.shape[0]
    cap = 10 * n if cfg.max_iters is None else cfg.max_iters
    defl = basis is not None and basis.k > 0
    if defl:
        low, w, aw = basis.factored(be), basis.w, basis.aw
    log = Log()
    nb = float(np.sqrt(b @ b))
    if nb == 0.0:
        log.r.append(np.zeros(n))
        return np.zeros(n), Report(0, [0.0], True, time.perf_counter() - t_start, "converged"), log
    x = x0.copy()
    r = b - kern.matvec(a, x)
    if defl:
        mu = chol_solve(low, aw.T @ r, be)
        p = r - w @ mu
    else:
        mu, p = None, r.copy()
    rr = float(r @ r)
    rel = np.sqrt(rr) / nb
    hist = [rel]
    log.r.append(r.copy())
    it = 0
    while rel > cfg.tol and it < cap:
        if it < cfg.ell:
            log.p.append(p.copy())
            if defl:
                log.mu.append(mu.copy())
        ap = kern.matvec(a, p)
        d = float(p @ ap)
        if d <= 0.0:
            raise OBreakdown(it)
        alpha = rr / d
        x += alpha * p
        it += 1
        if cfg.recompute_residual_every and it % cfg.recompute_residual_every == 0:
            r = b - kern.matvec(a, x)
        else:
            r = r - alpha * ap
        rr_next = float(r @ r)
        beta = rr_next / rr
        rel = np.sqrt(rr_next) / nb
        hist.append(rel)
        if it - 1 < cfg.ell:
            log.d.append(d)
            log.alpha.append(alpha)
            log.beta.append(beta)
            log.r.append(r.copy())
        if defl:
            mu = chol_solve(low, aw.T @ r, be)
            p = beta * p + r - w @ mu
        else:
            p = r + beta * p
        rr = rr_next
    ok = rel <= cfg.tol
    rep = Report(it, hist, ok, time.perf_counter() - t_start, "converged" if ok else "max_iters")
    return x, rep, log


def cg_solve(a, b, x0=None, cfg=None, be="compiled"):
    """solvers.py:207-219."""
    cfg = cfg or Cfg()
    b = _vec(b)
    x0 = np.zeros(b.shape[0]) if x0 is None else x0
    t0 = time.perf_counter()
    a, b, x0 = _system(a, b, x0)
    return krylov_loop(a, b, x0, None, cfg, t0, be)


def deflated_cg_solve(a, b, x_prev, basis, cfg=None, be="compiled"):
    """solvers.py:222-239 (warm start uses W', the loop AW')."""
    cfg = cfg or Cfg()
    t0 = time.perf_counter()
    a, b, x_prev = _system(a, b, x_prev)
    if basis.k == 0:
        return krylov_loop(a, b, x_prev, None, cfg, t0, be)
    if basis.w.shape[0] != b.shape[0]:
        raise ODimensionMismatch(f"basis rows {basis.w.shape[0]} vs system size {b.shape[0]}")
    low = basis.factored(be)
    r_prev = b - backend(be).matvec(a, x_prev)
    x0 = x_prev + basis.w @ chol_solve(low, basis.w.T @ r_prev, be)
    return krylov_loop(a, b, x0, basis, cfg, t0, be)


def deflation_project(a, basis, v, be="compiled"):
    """solvers.py:242-256."""
    a, v = _mat(a), _vec(v)
    if basis.k == 0:
        return v.copy()
    return v - basis.aw @ chol_solve(basis.factored(be), basis.w.T @ v, be)


# --------------------------------------------------------------------------
# recycling (recycle.py)
# --------------------------------------------------------------------------


def _prune_factor(w, aw, be):
    """recycle.py:66-77: drop the failing-pivot column until W'AW factors."""
    while True:
        if w.shape[1] == 0:
            raise OBasisDeficient(0)
        gram = w.T @ aw
        gram = 0.5 * (gram + gram.T)
        try:
            return w, aw, chol_factor(gram, be=be)
        except ONotPositiveDefinite as exc:
            w = np.delete(w, exc.pivot_index, axis=1)
            aw = np.delete(aw, exc.pivot_index, axis=1)


def refresh_basis(a_next, w, be="compiled"):
    """recycle.py:80-92."""
    a_next = check_symmetric(a_next)
    w = _mat(w)
    if w.shape[1] == 0:
        return Basis(w, w.copy(), np.empty((0, 0)))
    aw = backend(be).gemm(a_next, w)
    w, aw, low = _prune_factor(w, aw, be)
    return Basis(w, aw, low)


@dataclass
class Ritz:
    """RitzExtraction (recycle.py:31-46)."""

    theta: np.ndarray
    u: np.ndarray
    z: np.ndarray
    w_next: np.ndarray
    aw_next: np.ndarray
    selection: str


def harmonic_ritz(log, prev, k, selection="smallest", be="compiled"):
    """recycle.py:95-159."""
    if selection not in ("smallest", "largest"):
        raise ValueError(f"unknown selection {selection!r}")
    m = len(log.p)
    kp = prev.k if prev is not None else 0
    total = kp + m
    if k > total:
        raise OBasisDeficient(total)
    n = log.r[0].shape[0]
    if k == 0:
        e = np.empty((n, 0))
        return Ritz(np.empty(0), np.empty((total, 0)), e, e, e.copy(), selection)
    z = np.empty((n, total))
    az = np.empty((n, total))
    for j in range(kp):
        z[:, j] = prev.w[:, j]
        az[:, j] = prev.aw[:, j]
    for j in range(m):
        z[:, kp + j] = log.p[j]
        az[:, kp + j] = (log.r[j] - log.r[j + 1]) / log.alpha[j]
    nrm = np.linalg.norm(z, axis=0)
    keep = nrm > 0.0
    z = z[:, keep] / nrm[keep]
    az = az[:, keep] / nrm[keep]
    while True:
        if z.shape[1] < k:
            raise OBasisDeficient(z.shape[1])
        f = az.T @ z
        f = 0.5 * (f + f.T)
        g = az.T @ az
        g = 0.5 * (g + g.T)
        try:
            vals, vecs = gen_sym_eigen(g, f, be=be)
            break
        except ONotPositiveDefinite as exc:
            z = np.delete(z, exc.pivot_index, axis=1)
            az = np.delete(az, exc.pivot_index, axis=1)
    sel = np.arange(k) if selection == "smallest" else np.arange(vals.shape[0] - k, vals.shape[0])
    theta = vals[sel].copy()
    u = vecs[:, sel].copy()
    for j in range(k):
        scale = float(np.linalg.norm(z @ u[:, j]))
        if scale > 0.0:
            u[:, j] /= scale
    z, az, u = np.ascontiguousarray(z), np.ascontiguousarray(az), np.ascontiguousarray(u)
    kern = backend(be)
    return Ritz(theta, u, z, kern.gemm(z, u), kern.gemm(az, u), selection)


@dataclass
class Sequence:
    """SequenceState (recycle.py:49-63)."""

    k: int
    cfg: Cfg = field(default_factory=Cfg)
    selection: str = "smallest"
    basis: Basis | None = None
    x_last: np.ndarray | None = None
    history: list = field(default_factory=list)


def solve_next(state, a, b, be="compiled"):
    """recycle.py:162-203 (BasisDeficient swallowed in refresh and extraction)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x_prev = state.x_last if state.x_last is not None else np.zeros(b.shape[0])
    used = None
    if state.basis is not None and state.basis.k > 0:
        try:
            used = refresh_basis(a, state.basis.w, be)
        except OBasisDeficient:
            used = None
    if used is not None:
        x, rep, log = deflated_cg_solve(a, b, x_prev, used, state.cfg, be)
    else:
        x, rep, log = cg_solve(a, b, x_prev, state.cfg, be)
    nxt = None
    if state.k > 0:
        try:
            ext = harmonic_ritz(log, used, state.k, state.selection, be)
            if ext.w_next.shape[1] > 0:
                nxt = Basis(ext.w_next, ext.aw_next)
        except OBasisDeficient:
            nxt = None
    return x, replace(state, basis=nxt, x_last=x, history=state.history + [rep])


# --------------------------------------------------------------------------
# GP classification, Laplace approximation (gpc.py)
# --------------------------------------------------------------------------


def rbf_kernel(x, signal_sd=1.0, lengthscale=1.0, jitter=None, be="compiled"):
    """gpc.py:82-98."""
    x = _mat(x)
    if not np.all(np.isfinite(x)):
        raise ValueError("data matrix contains non-finite entries")
    var = signal_sd**2
    jitter = 1e-8 * var if jitter is None else jitter
    if jitter < 0.0:
        raise ValueError("jitter must be non-negative")
    return backend(be).rbf_gram(x, var, 1.0 / (2.0 * lengthscale**2), float(jitter))


def sigmoid(z):
    """Two-branch logistic (gpc.py:126-132)."""
    out = np.empty_like(z)
    pos = z >= 0.0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def likelihood_derivs(f, y):
    """gpc.py:142-157."""
    f = _vec(f)
    y = np.asarray(y, dtype=np.float64)
    loglik = float(-np.sum(np.logaddexp(0.0, -y * f)))
    pi = sigmoid(f)
    return loglik, (y + 1.0) * 0.5 - pi, pi * sigmoid(-f)


@dataclass
class NewtonStep:
    """NewtonRecord (gpc.py:68-79)."""

    newton_iter: int
    psi: float
    loglik: float
    solver_iterations: int | None
    rel_residual: float
    solve_time_s: float
    residual_history: list
    f: np.ndarray


def laplace_newton(k_matrix, y, solver="cholesky", cfg=None, newton_tol=1.0, max_newton=30, k=8,
                   selection="largest", be="compiled", max_steps_timed=None):
    """gpc.py:160-291 (make_state, build_newton_system, newton_update,
    psi_objective and the driver).  ``max_steps_timed`` (bench sampling only)
    stops after that many Newton steps."""
    if solver not in ("cholesky", "cg", "defcg"):
        raise ValueError(f"unknown solver {solver!r}")
    kern = backend(be)
    cfg = cfg or Cfg()
    kmat = _mat(k_matrix)
    y = np.asarray(y, dtype=np.float64)
    n = y.shape[0]
    f = np.zeros(n)
    a = np.zeros(n)
    loglik, grad, h = likelihood_derivs(f, y)

    def psi_of(f, a, loglik):
        err = float(np.linalg.norm(f - kern.matvec(kmat, a)))
        if err > 1e-8 * float(np.linalg.norm(f)):
            raise OStateInconsistent(f"||f - K a|| = {err:g}")
        return loglik - 0.5 * float(f @ a)

    psi_prev = psi_of(f, a, loglik)
    steps = []
    seq = Sequence(k=k, cfg=cfg, selection=selection)
    x_prev = np.zeros(n)
    for it in range(1, max_newton + 1):
        s = np.sqrt(h)
        amat = kmat * np.outer(s, s)
        idx = np.arange(n)
        amat[idx, idx] += 1.0
        inner = h * f + grad
        b = s * kern.matvec(kmat, inner)
        t0 = time.perf_counter()
        if solver == "cholesky":
            x = chol_solve(chol_factor(amat, be=be), b, be)
            dt = time.perf_counter() - t0
            its, hist = None, []
            nb = float(np.linalg.norm(b))
            res = float(np.linalg.norm(b - kern.matvec(amat, x)))
            rel = res / nb if nb > 0.0 else 0.0
        elif solver == "cg":
            x, rep, _ = cg_solve(amat, b, x_prev, cfg, be)
            dt = time.perf_counter() - t0
            its, hist, rel = rep.iterations, rep.residual_history, rep.residual_history[-1]
        else:
            x, seq = solve_next(seq, amat, b, be)
            dt = time.perf_counter() - t0
            rep = seq.history[-1]
            its, hist, rel = rep.iterations, rep.residual_history, rep.residual_history[-1]
        inner = h * f + grad
        a = inner - np.sqrt(h) * x
        f = kern.matvec(kmat, a)
        loglik, grad, h = likelihood_derivs(f, y)
        psi = psi_of(f, a, loglik)
        steps.append(NewtonStep(it, psi, loglik, its, rel, dt, list(hist), f.copy()))
        if psi < psi_prev - 1e-6:
            raise ONoProgress(f"objective fell from {psi_prev:.9g} to {psi:.9g} at iteration {it}")
        if psi - psi_prev < newton_tol:
            break
        if max_steps_timed is not None and it >= max_steps_timed:
            break
        psi_prev = psi
        x_prev = x
    return f, a, steps


# --------------------------------------------------------------------------
# synthetic inputs of BASELINE.json's configs
# --------------------------------------------------------------------------


def gpc_inputs(n, d, seed=0):
    """X ~ N(0, I_d) drawn first, then noise; y = sign(sum sin(2x) + 0.1 noise), sign(0) -> +1."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d))
    noise = rng.standard_normal(n)
    t = np.sin(2.0 * x).sum(axis=1) + 0.1 * noise
    y = np.where(t >= 0.0, 1.0, -1.0)
    return x, y


def sweep_inputs(n, d=8, seed=0):
    """Config 4: X ~ U[-1,1]^d, y = sum sin(3x) + 0.05 noise."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1.0, 1.0, (n, d))
    noise = rng.standard_normal(n)
    return x, np.sin(3.0 * x).sum(axis=1) + 0.05 * noise
