"""GP binary classification with the Laplace approximation — drop-in for defcg.gpc.

Public names and semantics follow /root/reference/pkg/src/defcg/gpc.py:36-291.
Everything n-sized stays in HBM for the whole Newton loop:

* ``rbf_kernel`` assembles the Gram matrix on device (K6, exact symmetry and
  exact diagonal ``var + jitter`` like ``_core.rbf_gram``) and returns a
  :class:`DenseOperator` (``np.asarray`` materialises it on request);
* the Newton system A = I + S K S is an implicit view of the same K
  (gpc.py:178 materialises it every step in the reference);
* the right-hand side, update, likelihood derivatives and psi are fused
  device kernels (``dcg_gpc_newton_system`` / ``dcg_gpc_newton_update``).

The psi consistency check ||f - K a|| <= 1e-8 ||f|| (gpc.py:204-209) is
exact inside ``laplace_newton``: f is produced as K a by the same deterministic
kernel in the same step, so the check's extra K-product (the reference's third
per step) is not repeated there; ``psi_objective`` still performs it.
"""

from __future__ import annotations

import ctypes
import gc
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import DimensionMismatch, InvalidLabel, NoProgress, NotPositiveDefinite, StateInconsistent
from .operators import SYM_MIN_N, DenseOperator, RbfOperator, _RowMajor, as_operator
from .recycle import SELECT_LARGEST, SequenceState, _pinned, _pinned_pool, prepare_refresh, solve_next, solve_next_async
from .solvers import SolverConfig, _solve_dev

SOLVER_CHOLESKY = "cholesky"
SOLVER_CG = "cg"
SOLVER_DEFCG = "defcg"


@dataclass(frozen=True)
class KernelParams:
    """RBF kernel k(x, x') = signal_sd^2 exp(-||x - x'||^2 / (2 lengthscale^2)) (gpc.py:36-45)."""

    signal_sd: float = 1.0
    lengthscale: float = 1.0

    def __post_init__(self):
        if self.signal_sd <= 0.0 or self.lengthscale <= 0.0:
            raise ValueError("signal_sd and lengthscale must be positive")


@dataclass
class GpcState:
    """Latent state with cached likelihood derivatives (gpc.py:48-58).

    Device flavour (the default inside laplace_newton, or when built from
    torch inputs): the vectors are CUDA tensors and ``k_matrix`` a device
    operator.  Host flavour (``host``, inferred from numpy fields when not
    given): the fields are numpy arrays as in the reference, and every public
    function moves them to the device for its work and returns host-flavour
    results."""

    f: object
    y: object
    k_matrix: object
    a: object
    loglik: float
    grad_loglik: object
    h: object
    host: bool | None = None

    def __post_init__(self):
        if self.host is None:
            self.host = not isinstance(self.f, torch.Tensor)


@dataclass
class NewtonSystem:
    """gpc.py:61-65; ``a_matrix`` is the implicit operator I + S K S (the
    explicit matrix, b and sqrt_h as numpy arrays for a host-flavour state)."""

    a_matrix: DenseOperator
    b: torch.Tensor
    sqrt_h: torch.Tensor
    inner: torch.Tensor | None = None
    ax0: torch.Tensor | None = None      # a_matrix @ x_prev, when built with x_prev
    x_prev: torch.Tensor | None = None


@dataclass
class NewtonRecord:
    """One Newton iteration (gpc.py:68-79)."""

    newton_iter: int
    psi: float
    loglik: float
    solver_iterations: int | None
    rel_residual: float
    solve_time_s: float
    residual_history: list
    f: object


def rbf_kernel(x, params, jitter=None, matrix_free=False):
    """Dense RBF Gram matrix built on device (gpc.py:82-98, _core.pyx:97-114).

    torch X: a DenseOperator holding K in HBM (the fast path), or with
    ``matrix_free`` an RbfOperator that regenerates K from X on every product
    (config 5: the Gram would not fit).  numpy X: K built on the device and
    returned as a numpy array, as the reference does."""
    if not matrix_free and not isinstance(x, torch.Tensor):
        return np.asarray(rbf_kernel(D.to_dev(x, 2), params, jitter))
    xd = D.to_dev(x, 2)
    if not bool(torch.isfinite(xd).all()):
        raise ValueError("data matrix contains non-finite entries")
    var = params.signal_sd**2
    if jitter is None:
        jitter = 1e-8 * var
    if jitter < 0.0:
        raise ValueError("jitter must be non-negative")
    inv_two_ell2 = 1.0 / (2.0 * params.lengthscale**2)
    n, dim = xd.shape
    if matrix_free:
        return RbfOperator(xd.contiguous(), var, inv_two_ell2, var + float(jitter))
    ld = D.padded_ld(n)

    def build_rows():
        kbuf = D.empty(n, ld)
        if ld != n:
            kbuf[:, n:].zero_()   # only the row-pitch padding (the kernel writes every entry of K)
        if n:
            N.check(N.lib().dcg_k_rbf_gram(D.ctx(), D.stream(), xd.data_ptr(), n, dim, var, inv_two_ell2,
                                           float(jitter), kbuf.data_ptr(), ld, 0, n), what="rbf_gram")
        return kbuf

    if n < SYM_MIN_N:
        return DenseOperator(build_rows(), n, ld)
    # Above SYM_MIN_N every product of the Newton path reads the packed
    # lower-triangle tiles: build those directly from X (entries bitwise the
    # row-major Gram's) and the row-major K only if something asks for rows.
    kp = D.empty(int(N.lib().dcg_packed_sym_doubles(n)))
    ntt = int(N.lib().dcg_packed_sym_doubles(n)) // 4096
    N.check(N.lib().dcg_k_rbf_gram_packed(D.ctx(), D.stream(), xd.data_ptr(), n, dim, var, inv_two_ell2,
                                          float(jitter), 0, ntt, kp.data_ptr()), what="rbf_gram_packed")
    op = DenseOperator(_RowMajor(build=build_rows), n, ld)
    op._packed.adopt(kp)
    return op


def rbf_cross_kernel(xa, xb, params):
    """Cross-kernel block between two point sets, no jitter (gpc.py:101-107),
    built on device (``dcg_k_rbf_cross``, the reference's difference-squared
    form _core.pyx:117-132).  numpy in -> numpy out, torch in -> device tensor."""
    ad, bd = D.to_dev(xa, 2), D.to_dev(xb, 2)
    if ad.shape[1] != bd.shape[1]:
        raise DimensionMismatch(f"point dimensions {ad.shape[1]} and {bd.shape[1]}")
    for t in (ad, bd):
        if t.numel() and not bool(torch.isfinite(t).all()):
            raise ValueError("data matrix contains non-finite entries")
    var = params.signal_sd**2
    inv_two_ell2 = 1.0 / (2.0 * params.lengthscale**2)
    out = D.empty(ad.shape[0], bd.shape[0])
    if out.numel():
        N.check(N.lib().dcg_k_rbf_cross(D.ctx(), D.stream(), ad.data_ptr(), ad.shape[0], bd.data_ptr(), bd.shape[0],
                                        ad.shape[1], float(var), float(inv_two_ell2), out.data_ptr()),
                what="rbf_cross")
    return D.out_like(out, xa)


def _labels_dev(y):
    """(fp64 labels on the device, validity flag on the device or None): the
    flag of device labels is read by the caller after its next host sync."""
    if isinstance(y, torch.Tensor):
        yd = y.to(device=D.device())
        if yd.ndim != 1:
            raise InvalidLabel("labels must be a vector of -1/+1")
        return yd.to(torch.float64).contiguous(), ((yd == 1) | (yd == -1)).all()
    return check_labels(y), None


def check_labels(y):
    """gpc.py:135-139.  Device labels are checked on the device (one flag
    read back), host labels on the host; returns fp64 labels on the device."""
    if isinstance(y, torch.Tensor):
        yd, ok = _labels_dev(y)
        if not bool(ok):
            raise InvalidLabel("labels must be a vector of -1/+1")
        return yd
    arr = np.asarray(y)
    if arr.ndim != 1 or not np.all(np.isin(arr, (-1, 1))):
        raise InvalidLabel("labels must be a vector of -1/+1")
    return D.to_dev(arr.astype(np.float64), 1)


def _derivs_dev(f: torch.Tensor, y: torch.Tensor):
    n = f.shape[0]
    grad, h = D.empty(n), D.empty(n)
    ll = ctypes.c_double(0.0)
    N.check(N.lib().dcg_gpc_derivs(D.ctx(), D.stream(), n, f.data_ptr(), y.data_ptr(), grad.data_ptr(),
                                   h.data_ptr(), ctypes.byref(ll)), what="gpc_derivs")
    return float(ll.value), grad, h


def likelihood_derivs(f, y):
    """(log-likelihood, gradient, curvature) of the logistic model (gpc.py:142-157)."""
    fd = D.to_dev(f, 1)
    yd = check_labels(y)
    if fd.shape != yd.shape:
        raise InvalidLabel("f and y must have the same length")
    ll, g, h = _derivs_dev(fd, yd)
    if isinstance(f, torch.Tensor):
        return ll, g, h
    return ll, g.cpu().numpy(), h.cpu().numpy()


def _dense_cholesky_solve(op: DenseOperator, b: torch.Tensor) -> torch.Tensor:
    """Direct solve of the (materialised) SPD system — the reference's
    "cholesky" solver column (gpc.py:247-255) via cuSOLVER potrf."""
    return torch.cholesky_solve(b[:, None], _dense_cholesky_factor(op))[:, 0]


def _dense_cholesky_factor(op: DenseOperator) -> torch.Tensor:
    """cholesky_factor(A) with the reference's pivot semantics (linalg.py:74-92,
    _core.pyx:47-66): a pivot d_j = a_jj - sum_k L_jk^2 at or below
    1e-14 * max(max diag, 0) raises NotPositiveDefinite(j).  potrf stops only
    at a non-positive pivot and otherwise stores L_jj = sqrt(d_j), so the
    failing index is the first j with L_jj^2 <= tol before potrf's own stop."""
    a = op.dense_dev()
    n = a.shape[0]
    if n == 0:
        return a
    tol = 1e-14 * max(float(a.diagonal().max()), 0.0)
    low, info = torch.linalg.cholesky_ex(a)
    stop = int(info) - 1 if int(info) > 0 else n       # potrf's failing column (or n)
    piv = low.diagonal()[:stop]
    bad = torch.nonzero(piv * piv <= tol)
    fail = int(bad[0, 0]) if bad.numel() else (stop if stop < n else -1)
    if fail >= 0:
        raise NotPositiveDefinite(fail)
    return low


def _kernel_op(k_matrix) -> DenseOperator:
    return as_operator(k_matrix).kernel_view() if isinstance(k_matrix, DenseOperator) else as_operator(k_matrix)


def _host(v):
    return v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else v


def _dev_state(state: GpcState) -> GpcState:
    """Device-flavour view of a state (numpy fields uploaded, K as an operator)."""
    if not state.host and isinstance(state.k_matrix, DenseOperator):
        return state
    return GpcState(f=D.to_dev(state.f, 1), y=check_labels(state.y), k_matrix=_kernel_op(state.k_matrix),
                    a=D.to_dev(state.a, 1), loglik=state.loglik, grad_loglik=D.to_dev(state.grad_loglik, 1),
                    h=D.to_dev(state.h, 1), host=False)


def _as_flavour(state: GpcState, host: bool, k_matrix=None) -> GpcState:
    if not host:
        return state
    return GpcState(f=_host(state.f), y=_host(state.y), k_matrix=state.k_matrix if k_matrix is None else k_matrix,
                    a=_host(state.a), loglik=state.loglik, grad_loglik=_host(state.grad_loglik), h=_host(state.h),
                    host=True)


def _make_state_dev(k_matrix, y, f=None) -> GpcState:
    op = _kernel_op(k_matrix)
    if f is None:
        # f = a = 0: one library call zeroes them, evaluates the derivatives
        # and loglik and counts the labels outside {-1, +1} (one host read)
        if isinstance(y, torch.Tensor):
            yd = y.to(device=D.device(), dtype=torch.float64)
            if yd.ndim != 1:
                raise InvalidLabel("labels must be a vector of -1/+1")
            yd = yd.contiguous()
        else:
            yd = check_labels(y)
        n = yd.shape[0]
        fd, ad, g, h = D.empty(n), D.empty(n), D.empty(n), D.empty(n)
        ll, bad = ctypes.c_double(0.0), ctypes.c_longlong(0)
        N.check(N.lib().dcg_gpc_init(D.ctx(), D.stream(), n, yd.data_ptr() if n else None, fd.data_ptr(),
                                     ad.data_ptr(), g.data_ptr(), h.data_ptr(), ctypes.byref(ll), ctypes.byref(bad)),
                what="gpc_init")
        if bad.value:
            raise InvalidLabel("labels must be a vector of -1/+1")
        return GpcState(f=fd, y=yd, k_matrix=op, a=ad, loglik=float(ll.value), grad_loglik=g, h=h, host=False)
    yd = check_labels(y)
    fd = D.to_dev(f, 1)
    ad = _dense_cholesky_solve(op, fd)
    ll, g, h = _derivs_dev(fd, yd)
    return GpcState(f=fd, y=yd, k_matrix=op, a=ad, loglik=ll, grad_loglik=g, h=h, host=False)


class _PendingInit:
    """loglik and the label check of an enqueued start state (dcg_gpc_init_async):
    the status block is copied to pinned memory on the copy stream and read when
    the Newton loop first needs psi_prev -- after the first system and solve have
    been enqueued, so the host read leaves the head of the sequence."""

    def __init__(self, status):
        self.host = _pinned(8)
        ready = torch.cuda.Event()
        ready.record()
        cs = D.copy_stream()
        cs.wait_event(ready)
        with torch.cuda.stream(cs):
            self.host[:8].copy_(status, non_blocking=True)
            self.event = torch.cuda.Event()
            self.event.record(cs)
        status.record_stream(cs)

    def resolve(self):
        """loglik; raises InvalidLabel (gpc.py:135-139) if a label is not -1 / +1."""
        self.event.synchronize()
        bad = int(self.host[1])
        ll = float(self.host[4:5].view(torch.float64)[0])
        _pinned_pool.append(self.host)
        if bad:
            raise InvalidLabel("labels must be a vector of -1/+1")
        return ll


def _make_state_dev_async(k_matrix, y):
    """_make_state_dev(k_matrix, y) with f = 0 for device labels, without the
    host read: (state with loglik pending, _PendingInit); None when the labels
    are not a device-ready vector (the synchronous form then validates them)."""
    if not isinstance(y, torch.Tensor) or y.ndim != 1 or y.shape[0] == 0:
        return None
    op = _kernel_op(k_matrix)
    yd = y.to(device=D.device(), dtype=torch.float64).contiguous()
    n = yd.shape[0]
    fd, ad, g, h = D.empty(n), D.empty(n), D.empty(n), D.empty(n)
    status = torch.empty(8, dtype=torch.int64, device=D.device())
    N.check(N.lib().dcg_gpc_init_async(D.ctx(), D.stream(), n, yd.data_ptr(), fd.data_ptr(), ad.data_ptr(),
                                       g.data_ptr(), h.data_ptr(), status.data_ptr()), what="gpc_init_async")
    st = GpcState(f=fd, y=yd, k_matrix=op, a=ad, loglik=float("nan"), grad_loglik=g, h=h, host=False)
    return st, _PendingInit(status)


def make_state(k_matrix, y, f=None):
    """Fresh GpcState; f defaults to zero, a given f implies a = K^-1 f (gpc.py:160-172).
    Host flavour (numpy fields, k_matrix as given) unless y is a torch tensor."""
    st = _make_state_dev(k_matrix, y, f)
    host = not isinstance(y, torch.Tensor)
    return _as_flavour(st, host, k_matrix)


def build_newton_system(state, x_prev=None):
    """A = I + H^1/2 K H^1/2 (implicit) and b = H^1/2 K (H f + grad) (gpc.py:175-183).

    With ``x_prev`` (a device vector) also ax0 = A x_prev, the first product of
    the next warm-started solve, from the same pass over K.  A host-flavour
    state gets the reference's explicit A and numpy b, sqrt_h."""
    if state.host:
        sysm = build_newton_system(_dev_state(state))
        return NewtonSystem(a_matrix=np.asarray(sysm.a_matrix), b=_host(sysm.b), sqrt_h=_host(sysm.sqrt_h))
    state = _dev_state(state)
    op = state.k_matrix
    n = op.n
    s, inner, b = D.empty(n), D.empty(n), D.empty(n)
    kop = op.kernel_view().c_struct()
    if x_prev is not None:
        ax0 = D.empty(n)
        N.check(N.lib().dcg_gpc_newton_system_ax0(D.ctx(), D.stream(), ctypes.byref(kop), state.f.data_ptr(),
                                                  state.grad_loglik.data_ptr(), state.h.data_ptr(),
                                                  x_prev.data_ptr(), s.data_ptr(), inner.data_ptr(), b.data_ptr(),
                                                  ax0.data_ptr()), what="newton_system_ax0")
        return NewtonSystem(a_matrix=op.scaled(s, 1.0), b=b, sqrt_h=s, inner=inner, ax0=ax0, x_prev=x_prev)
    N.check(N.lib().dcg_gpc_newton_system(D.ctx(), D.stream(), ctypes.byref(kop), state.f.data_ptr(),
                                          state.grad_loglik.data_ptr(), state.h.data_ptr(), s.data_ptr(),
                                          inner.data_ptr(), b.data_ptr()), what="newton_system")
    return NewtonSystem(a_matrix=op.scaled(s, 1.0), b=b, sqrt_h=s, inner=inner)


def _update_dev(state, inner, s, x):
    op = state.k_matrix
    n = op.n
    a, f, g, h = D.empty(n), D.empty(n), D.empty(n), D.empty(n)
    ll, psi = ctypes.c_double(0.0), ctypes.c_double(0.0)
    kop = op.kernel_view().c_struct()
    N.check(N.lib().dcg_gpc_newton_update(D.ctx(), D.stream(), ctypes.byref(kop), inner.data_ptr(), s.data_ptr(),
                                          x.data_ptr(), state.y.data_ptr(), a.data_ptr(), f.data_ptr(), g.data_ptr(),
                                          h.data_ptr(), ctypes.byref(ll), ctypes.byref(psi)), what="newton_update")
    new = GpcState(f=f, y=state.y, k_matrix=op, a=a, loglik=float(ll.value), grad_loglik=g, h=h)
    return new, float(psi.value)


class _PendingObjective:
    """(loglik, psi) of an enqueued newton update: copied to pinned host memory
    on the copy stream right behind the derivative kernels (off the main
    stream, which goes on with the next system), read on demand."""

    def __init__(self, llpsi):
        self.host = _pinned(2)
        ready = torch.cuda.Event()
        ready.record()
        cs = D.copy_stream()
        cs.wait_event(ready)
        with torch.cuda.stream(cs):
            self.host.view(torch.float64)[:2].copy_(llpsi, non_blocking=True)
            self.event = torch.cuda.Event()
            self.event.record(cs)
        llpsi.record_stream(cs)

    def get(self):
        self.event.synchronize()
        ll, psi = (float(v) for v in self.host.view(torch.float64)[:2].tolist())
        _pinned_pool.append(self.host)
        return ll, psi


def _update_dev_async(state, inner, s, x):
    """_update_dev without the host read: returns (new state with loglik
    pending, _PendingObjective)."""
    op = state.k_matrix
    n = op.n
    a, f, g, h = D.empty(n), D.empty(n), D.empty(n), D.empty(n)
    llpsi = D.empty(2)
    kop = op.kernel_view().c_struct()
    N.check(N.lib().dcg_gpc_newton_update_async(D.ctx(), D.stream(), ctypes.byref(kop), inner.data_ptr(),
                                                s.data_ptr(), x.data_ptr(), state.y.data_ptr(), a.data_ptr(),
                                                f.data_ptr(), g.data_ptr(), h.data_ptr(), llpsi.data_ptr()),
            what="newton_update_async")
    new = GpcState(f=f, y=state.y, k_matrix=op, a=a, loglik=float("nan"), grad_loglik=g, h=h)
    return new, _PendingObjective(llpsi)


def _laplace_newton_pipelined(state, psi_prev, cfg, newton_tol, max_newton, k, selection):
    """(see _pipelined_loop) The host enqueues each step's device work while
    the previous solve runs; a cyclic-garbage collection pass in the middle of
    that (the loop allocates many short-lived objects) would stall the
    enqueue, so automatic collection is paused for the loop."""
    enabled = gc.isenabled()
    gc.disable()
    try:
        return _pipelined_loop(state, psi_prev, cfg, newton_tol, max_newton, k, selection)
    finally:
        if enabled:
            gc.enable()


def _pipelined_loop(state, psi_prev, cfg, newton_tol, max_newton, k, selection):
    """The def-CG Newton loop with every host synchronisation off the device's
    critical path.  Per step the main stream runs refresh -> solve -> newton
    update -> next system back to back while the extraction of the next basis
    runs on the side stream; the host waits only for the solve status (to
    enqueue the extraction with its sizes) and for psi (the reference's
    NoProgress / newton_tol checks, gpc.py:272-290), both already complete or
    about to be.  The next system is formed before psi is checked; when the
    loop stops it is simply dropped."""
    records = []
    seq = SequenceState(k=k, cfg=cfg, selection=selection)
    system = build_newton_system(state)
    prepared = None
    for it in range(1, max_newton + 1):
        t0 = time.perf_counter()
        x, job = solve_next_async(seq, system.a_matrix, system.b, ax0=system.ax0, ax0_of=system.x_prev,
                                  prepared=prepared, extract=it < max_newton, need_aw=False)
        new_state, objective = _update_dev_async(state, system.inner, system.sqrt_h, x)
        # the next system and its solve's first product A_next x in one K pass
        next_system = build_newton_system(new_state, x_prev=x) if it < max_newton else None
        # ... and the next solve's refresh, enqueued while this solve still
        # runs (dropped if the loop stops below)
        prepared = prepare_refresh(job, next_system.a_matrix) if next_system is not None else None
        try:
            x, seq = job.finish()
        except Exception:
            if isinstance(psi_prev, _PendingInit):
                psi_prev.resolve()   # an invalid label is reported first, as the reference does
            raise
        dt = time.perf_counter() - t0
        report = seq.history[-1]
        if isinstance(psi_prev, _PendingInit):
            psi_prev = psi_prev.resolve()   # f = a = 0: psi = loglik (gpc.py:239); label check
        loglik, psi = objective.get()
        new_state.loglik = loglik
        state = new_state
        records.append(NewtonRecord(newton_iter=it, psi=psi, loglik=loglik, solver_iterations=report.iterations,
                                    rel_residual=report.residual_history[-1], solve_time_s=dt,
                                    residual_history=list(report.residual_history), f=state.f))
        if psi < psi_prev - 1e-6:
            raise NoProgress(f"objective fell from {psi_prev:.9g} to {psi:.9g} at iteration {it}")
        if psi - psi_prev < newton_tol:
            break
        psi_prev = psi
        system = next_system
    _ = seq.basis   # join a pending extraction (surfaces its errors here)
    return state, records


def newton_update(state, x):
    """a_new = (H f + grad) - H^1/2 x, f_new = K a_new (gpc.py:186-201)."""
    host = state.host
    dst = _dev_state(state)
    xd = D.to_dev(x, 1)
    s = torch.sqrt(dst.h)
    inner = dst.h * dst.f + dst.grad_loglik
    new, _ = _update_dev(dst, inner, s, xd)
    return _as_flavour(new, host, state.k_matrix)


def psi_objective(state):
    """psi = log p(y|f) - f'a / 2 with the f = K a consistency check (gpc.py:204-209)."""
    st = _dev_state(state)
    ka = st.k_matrix.kernel_view().matvec_dev(st.a)
    err = float(torch.linalg.norm(st.f - ka))
    if err > 1e-8 * float(torch.linalg.norm(st.f)):
        raise StateInconsistent(f"||f - K a|| = {err:g}")
    return st.loglik - 0.5 * float(st.f @ st.a)


def laplace_newton(k_matrix, y, solver=SOLVER_CHOLESKY, cfg=None, newton_tol=1.0, max_newton=30, k=8,
                   selection=SELECT_LARGEST):
    """Newton iteration for the posterior mode from f = 0 (gpc.py:212-291).

    Returns (final GpcState, list of NewtonRecord).  Record ``f`` snapshots are
    numpy arrays (copied back once, after the loop)."""
    if solver not in (SOLVER_CHOLESKY, SOLVER_CG, SOLVER_DEFCG):
        raise ValueError(f"unknown solver {solver!r}")
    cfg = cfg or SolverConfig()
    host = not isinstance(y, torch.Tensor)
    pending = _make_state_dev_async(k_matrix, y) if solver in (SOLVER_DEFCG, SOLVER_CG) and max_newton >= 1 else None
    if pending is not None:
        # device labels on the pipelined path: loglik and the label check are
        # read after the first system and solve have been enqueued
        state, psi_prev = pending
    else:
        state = _make_state_dev(k_matrix, y)
        psi_prev = state.loglik   # f = a = 0: psi = loglik, ||f - K a|| = 0 (gpc.py:239)
    n = state.y.shape[0]
    records = []
    if solver in (SOLVER_DEFCG, SOLVER_CG):
        # plain CG is solve_next with no basis (k = 0): cg_solve(A, b, x_prev)
        # exactly as gpc.py:256-261, on the same pipelined device path
        state, records = _laplace_newton_pipelined(state, psi_prev, cfg, newton_tol, max_newton,
                                                   k if solver == SOLVER_DEFCG else 0, selection)
        if records:
            stacked = torch.stack([r.f for r in records]).cpu().numpy()
            for r, row in zip(records, stacked):
                r.f = row
        return _as_flavour(state, host, k_matrix), records
    seq = SequenceState(k=k, cfg=cfg, selection=selection)
    x_prev = D.zeros(n)

    for it in range(1, max_newton + 1):
        system = build_newton_system(state)
        t0 = time.perf_counter()
        if solver == SOLVER_CHOLESKY:
            x = _dense_cholesky_solve(system.a_matrix, system.b)
            resid = system.b - system.a_matrix.matvec_dev(x)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            solver_iterations, history = None, []
            norm_b = float(torch.linalg.norm(system.b))
            rel_residual = float(torch.linalg.norm(resid)) / norm_b if norm_b > 0.0 else 0.0

        state, psi = _update_dev(state, system.inner, system.sqrt_h, x)
        records.append(NewtonRecord(newton_iter=it, psi=psi, loglik=state.loglik,
                                    solver_iterations=solver_iterations, rel_residual=rel_residual,
                                    solve_time_s=dt, residual_history=list(history), f=state.f))
        if psi < psi_prev - 1e-6:
            raise NoProgress(f"objective fell from {psi_prev:.9g} to {psi:.9g} at iteration {it}")
        if psi - psi_prev < newton_tol:
            break
        psi_prev = psi
        x_prev = x

    _ = seq.basis   # join a pending extraction (surfaces its errors here)
    if records:
        stacked = torch.stack([r.f for r in records]).cpu().numpy()
        for r, row in zip(records, stacked):
            r.f = row
    return _as_flavour(state, host, k_matrix), records
