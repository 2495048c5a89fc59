"""Subspace recycling — the drop-in for defcg.recycle.

``refresh_basis``, ``harmonic_ritz_extract``, ``SequenceState`` and
``solve_next`` keep the reference's names, defaults and semantics
(/root/reference/pkg/src/defcg/recycle.py:31-203), including the two places
where ``BasisDeficient`` is swallowed (recycle.py:178-179, 194-195) so the
sequence silently degrades to plain CG exactly when the reference does.
W, AW, the Krylov log and the warm start stay in HBM across the sequence:

  refresh   AW = A W in one pass over K on FP64 tensor cores, W'AW and the
            failing-pivot pruning Cholesky in one CTA      (dcg_refresh_basis)
  solve     the persistent CG / def-CG kernel              (dcg_solve)
  extract   Z = [W, P_m], AZ = [AW, (r_j - r_j+1)/alpha_j] normalised, the
            harmonic pencil F, G, pruning + Jacobi in one CTA, W_next = Z U
                                                           (dcg_ritz_extract)
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import BasisDeficient, DimensionMismatch
from .operators import DenseOperator, as_operator
from .solvers import TERM_CONVERGED, TERM_MAX_ITERS, KrylovLog, RecycleBasis, SolveReport, SolverConfig, _solve_dev

SELECT_SMALLEST = "smallest"
SELECT_LARGEST = "largest"


class RitzExtraction:
    """Harmonic Ritz values/vectors chosen for the next basis (recycle.py:31-46).

    Device tensors ``*_dev``; numpy views ``theta``, ``u``, ``z``, ``w_next``,
    ``aw_next`` materialise on access."""

    def __init__(self, theta, u, z, w_next, aw_next, selection):
        self.theta_dev, self.u_dev, self.z_dev = theta, u, z
        self.w_next_dev, self.aw_next_dev = w_next, aw_next
        self.selection = selection

    theta = property(lambda self: self.theta_dev.cpu().numpy())
    u = property(lambda self: self.u_dev.cpu().numpy())
    z = property(lambda self: self.z_dev.cpu().numpy())
    w_next = property(lambda self: self.w_next_dev.cpu().numpy())
    aw_next = property(lambda self: self.aw_next_dev.cpu().numpy())


class _PendingBasis:
    """A Ritz extraction enqueued on the side stream (dcg_ritz_extract_async).

    Resolved on first use: the current stream waits for the side stream's
    event, the 3-word device result is read, and the outcome maps to the next
    basis (ok), None (BasisDeficient, swallowed as in recycle.py:194-195) or
    the reference's exception (e.g. NoConvergence)."""

    def __init__(self, event, result, w_next, aw_next, keep_alive, tail=None):
        self.event = event
        self.result = result
        self.w_next = w_next
        self.aw_next = aw_next
        self.keep_alive = keep_alive   # inputs the side stream reads
        self.tail = tail               # enqueues the extraction's last stage on a given stream

    def join(self, stream):
        """Order `stream` after the extraction: wait for the side stream's
        event, then enqueue the extraction's tail (if split off) on `stream`."""
        stream.wait_event(self.event)
        if self.tail is not None:
            tail, self.tail = self.tail, None
            tail(stream)
            self.event = torch.cuda.Event()
            self.event.record(stream)

    def resolve(self):
        self.join(torch.cuda.current_stream())
        self.event.synchronize()
        status, info = (int(v) for v in self.result[:2].cpu().tolist())
        self.keep_alive = None
        if status == N.DCG_E_BASIS_DEFICIENT:
            return None
        N.check(status, info, "ritz_extract")
        if self.w_next.shape[1] == 0:
            return None
        nb = RecycleBasis.__new__(RecycleBasis)
        nb.w_dev, nb.aw_dev, nb.chol_dev = self.w_next, self.aw_next, None
        return nb


@dataclass
class SequenceState:
    """Carry-over between solves of a sequence (recycle.py:49-63).

    ``basis`` may hold an extraction still running on the side stream; reading
    the attribute waits for it."""

    k: int
    cfg: SolverConfig = field(default_factory=SolverConfig)
    selection: str = SELECT_SMALLEST
    basis: RecycleBasis | None = None
    x_last: object | None = None
    history: list = field(default_factory=list)

    def __getattribute__(self, name):
        value = object.__getattribute__(self, name)
        if name == "basis" and isinstance(value, _PendingBasis):
            value = value.resolve()
            object.__setattr__(self, "basis", value)
        return value


def _refresh_dev(op, w_dev: torch.Tensor) -> RecycleBasis:
    n, k = w_dev.shape
    if k == 0:
        return RecycleBasis(w_dev, w_dev.clone(), D.empty(0, 0))
    if op.n != n:
        raise DimensionMismatch(f"basis rows {n} vs operator size {op.n}")
    w_out, aw_out, chol = D.empty(n, k), D.empty(n, k), D.empty(k, k)
    kout, info = ctypes.c_longlong(k), ctypes.c_longlong(0)
    cop = op.c_struct(block_k=k) if isinstance(op, DenseOperator) else op.c_struct()
    rc = N.lib().dcg_refresh_basis(D.ctx(), D.stream(), ctypes.byref(cop), w_dev.data_ptr(), k, w_out.data_ptr(),
                                   aw_out.data_ptr(), chol.data_ptr(), ctypes.byref(kout), ctypes.byref(info))
    N.check(rc, info.value, "refresh_basis")
    kk = int(kout.value)
    basis = RecycleBasis.__new__(RecycleBasis)
    # the library writes the surviving columns compacted: n x kk row-major
    basis.w_dev = w_out.view(-1)[: n * kk].view(n, kk)
    basis.aw_dev = aw_out.view(-1)[: n * kk].view(n, kk)
    basis.chol_dev = chol.view(-1)[: kk * kk].view(kk, kk)
    return basis


def refresh_basis(a_next, w):
    """Rebuild a RecycleBasis for a new matrix: AW against a_next, W'AW
    factored with failing-pivot pruning (recycle.py:80-92).  Raises
    BasisDeficient(0) when nothing survives."""
    op = as_operator(a_next)
    if not isinstance(w, torch.Tensor):
        w = np.ascontiguousarray(w, dtype=np.float64)
    if w.ndim != 2:
        raise DimensionMismatch(f"expected a matrix, got ndim={w.ndim}")
    return _refresh_dev(op, D.to_dev(w, 2))


def _extract_dev(log: KrylovLog, prev: RecycleBasis | None, k: int, selection: str) -> RitzExtraction:
    if selection not in (SELECT_SMALLEST, SELECT_LARGEST):
        raise ValueError(f"unknown selection {selection!r}")
    m = log.stored_iterations
    kp = prev.k if prev is not None else 0
    total = kp + m
    if k > total:
        raise BasisDeficient(total)
    n = log.n
    if k == 0:
        e = D.empty(n, 0)
        return RitzExtraction(D.empty(0), D.empty(total, 0), e, e, e.clone(), selection)
    theta = D.empty(k)
    u = D.empty(total, k)
    z = D.empty(n, total)
    w_next, aw_next = D.empty(n, k), D.empty(n, k)
    t_out, info = ctypes.c_longlong(total), ctypes.c_longlong(0)
    clog = log.c_struct()
    cprev = prev.c_struct() if kp else None
    rc = N.lib().dcg_ritz_extract(D.ctx(), D.stream(), n, ctypes.byref(clog), m,
                                  ctypes.byref(cprev) if cprev is not None else None, k,
                                  N.DCG_SELECT_LARGEST if selection == SELECT_LARGEST else N.DCG_SELECT_SMALLEST,
                                  theta.data_ptr(), u.data_ptr(), z.data_ptr(), w_next.data_ptr(), aw_next.data_ptr(),
                                  ctypes.byref(t_out), ctypes.byref(info))
    N.check(rc, info.value, "ritz_extract")
    t = int(t_out.value)
    return RitzExtraction(theta, u.view(-1)[: t * k].view(t, k), z.view(-1)[: n * t].view(n, t), w_next, aw_next,
                          selection)


def _extract_async(log: KrylovLog, prev: RecycleBasis | None, k: int, selection: str,
                   after: "torch.cuda.Event | None" = None) -> "_PendingBasis | None":
    """Enqueue the extraction on the side stream (own context and workspace).
    The side stream waits for `after` (the solve) if given, else for
    everything enqueued on the main stream so far."""
    m = log.stored_iterations
    kp = prev.k if prev is not None else 0
    if k > kp + m:
        return None   # BasisDeficient, swallowed by solve_next
    n = log.n
    main = torch.cuda.current_stream()
    side = D.side_stream()
    if after is not None:
        side.wait_event(after)
    else:
        side.wait_stream(main)
    theta = D.empty(k)
    w_next, aw_next = D.empty(n, k), D.empty(n, k)
    result = torch.zeros(4, dtype=torch.int64, device=D.device())
    clog = log.c_struct()
    cprev = prev.c_struct() if kp else None
    _slot1_owner[D.device().index] = None   # the slot-1 workspace now holds this extraction's data
    with torch.cuda.stream(side):
        rc = N.lib().dcg_ritz_extract_async(D.ctx(1), side.cuda_stream, n, ctypes.byref(clog), m,
                                            ctypes.byref(cprev) if cprev is not None else None, k,
                                            N.DCG_SELECT_LARGEST if selection == SELECT_LARGEST
                                            else N.DCG_SELECT_SMALLEST,
                                            theta.data_ptr(), None, None, w_next.data_ptr(), aw_next.data_ptr(),
                                            result.data_ptr())
        N.check(rc, 0, "ritz_extract_async")
        event = torch.cuda.Event()
        event.record(side)
    return _PendingBasis(event, result, w_next, aw_next, (log, prev, theta))


# ---------------------------------------------------------------------------
# Pipelined sequence step (no host synchronisation between the extraction,
# the refresh and the solve).  solve_next's semantics are kept: the refresh
# uses the previous basis' W against the new operator, a BasisDeficient
# refresh (or a failed extraction) runs plain CG -- decided on the device:
# dcg_refresh_basis_async leaves the surviving column count in HBM and the
# solve kernel reads it -- and the next extraction uses the basis actually
# used.  The caller can enqueue independent work (the Newton update and the
# next system) between solve_next_async and finish().
# ---------------------------------------------------------------------------
_STATUS_WORDS = 8   # the 64-byte status block of dcg_solve_async

# Per device: the pending extraction whose intermediates the slot-1 context
# workspace currently holds (its split-off tail reads them at join time).
_slot1_owner: dict = {}


_pinned_pool: list = []


def _pinned(nwords):
    for i, t in enumerate(_pinned_pool):
        if t.numel() >= nwords:
            return _pinned_pool.pop(i)
    return torch.empty(max(nwords, 64), dtype=torch.int64, pin_memory=True)


_HIST_PREFIX = 1024   # residual-history entries copied back eagerly


class _AsyncSolve:
    """A refresh + solve (+ the next extraction) in flight.  The status block
    and a prefix of the residual history come back on the copy stream as soon
    as the solve ends, whatever the compute streams do next."""

    def __init__(self, state, x, log, hist, status, basis, event, ev_end, t0, cfg, pending, consumed=None,
                 combined=None):
        self.state, self.x, self.log, self.hist, self.status = state, x, log, hist, status
        self.basis, self.event, self.t0, self.cfg, self.pending = basis, event, t0, cfg, pending
        self.ev_end = ev_end
        # `consumed`: the result block of the extraction whose basis this solve
        # was handed (device side, a failed one degraded it to plain CG); read
        # back with the status so anything but BasisDeficient is raised
        self.consumed = consumed
        cs = D.copy_stream()
        cs.wait_event(self.ev_end)
        self.host = _pinned(_STATUS_WORDS + _HIST_PREFIX + 2)
        npre = min(_HIST_PREFIX, hist.shape[0])
        with torch.cuda.stream(cs):
            if combined is not None:
                # status words and history in one device buffer: one copy
                self.host[:_STATUS_WORDS + npre].view(torch.float64).copy_(combined[:_STATUS_WORDS + npre],
                                                                           non_blocking=True)
            else:
                self.host[:_STATUS_WORDS].copy_(status, non_blocking=True)
                self.host[_STATUS_WORDS:_STATUS_WORDS + npre].view(torch.float64).copy_(hist[:npre],
                                                                                        non_blocking=True)
            if consumed is not None:
                self.host[_STATUS_WORDS + _HIST_PREFIX:_STATUS_WORDS + _HIST_PREFIX + 2].copy_(consumed[:2],
                                                                                            non_blocking=True)
            self.done = torch.cuda.Event()
            self.done.record(cs)

    def finish(self):
        """Wait for the solve and build its report.  Returns (x, new SequenceState)."""
        self.done.synchronize()
        words = self.host[:_STATUS_WORDS].numpy().copy()
        if self.consumed is not None:
            # recycle.py:194-195 swallows only BasisDeficient; any other failure
            # of the extraction (e.g. NoConvergence of the pencil) propagates
            xst, xinfo = (int(v) for v in self.host[_STATUS_WORDS + _HIST_PREFIX:
                                                    _STATUS_WORDS + _HIST_PREFIX + 2].tolist())
            if xst not in (N.DCG_OK, N.DCG_E_BASIS_DEFICIENT):
                _pinned_pool.append(self.host)
                N.check(xst, xinfo, "ritz_extract")
        status = int(np.int32(words[0] & 0xFFFFFFFF))
        kused = int(words[0] >> 32)
        info = int(words[1])
        if status != N.DCG_OK:
            _pinned_pool.append(self.host)
            N.check(status, info, "solve")
        its, m = int(words[2]), int(words[3])
        rel = float(words[4:5].view(np.float64)[0])
        if its + 1 <= _HIST_PREFIX:
            history = self.host[_STATUS_WORDS:_STATUS_WORDS + its + 1].view(torch.float64).tolist()
        else:
            history = self.hist[: its + 1].cpu().tolist()
        _pinned_pool.append(self.host)
        conv = rel <= self.cfg.tol
        ms = self.event.elapsed_time(self.ev_end)
        rep = SolveReport(its, history, conv, time.perf_counter() - self.t0,
                          TERM_CONVERGED if conv else TERM_MAX_ITERS, float(ms))
        self.log.m, self.log.k = m, kused
        st = self.state
        return self.x, replace(st, basis=self.pending, x_last=self.x, history=st.history + [rep])


class _PreparedRefresh:
    """The refresh of the next solve (recycle.py:80-92 with the BasisDeficient
    rule of solve_next, recycle.py:178-179), enqueued ahead of time by
    prepare_refresh: the pending extraction's tail, A_next W_next, the pruned
    Gram factor.  solve_next_async uses it when it is handed the same basis
    object and the same operator."""

    def __init__(self, basis_obj, op, kmax, cb, kdev, bufs, valid):
        self.basis_obj, self.op, self.kmax, self.cb, self.kdev, self.bufs = basis_obj, op, kmax, cb, kdev, bufs
        self.valid = valid


def _enqueue_refresh(pending, op, n, main):
    """Refresh of the basis `pending` (a _PendingBasis, a RecycleBasis or None)
    for `op`, enqueued on `main`; returns (kmax, cb, kdev, bufs, valid), valid
    the pending extraction's device result block (or None)."""
    w_src, valid = None, None
    if isinstance(pending, _PendingBasis):
        w_src, valid = pending.w_next, pending.result
    elif pending is not None and pending.k > 0:
        w_src = pending.w_dev
    kmax = 0 if w_src is None else int(w_src.shape[1])
    cb, kdev, bufs = None, None, None
    if isinstance(pending, _PendingBasis) and not kmax:
        pending.join(main)
        pending.keep_alive = None
    if kmax:
        w_out, aw_out, chol = D.empty(n, kmax), D.empty(n, kmax), D.empty(kmax, kmax)
        kdev = torch.empty(1, dtype=torch.int64, device=D.device())
        cop = op.c_struct(block_k=kmax) if isinstance(op, DenseOperator) else op.c_struct()
        if isinstance(pending, _PendingBasis):
            pending.join(main)
            pending.keep_alive = None   # main-stream work is now ordered after the extraction
        N.check(N.lib().dcg_refresh_basis_async(D.ctx(), main.cuda_stream, ctypes.byref(cop), w_src.data_ptr(),
                                                kmax, valid.data_ptr() if valid is not None else None,
                                                w_out.data_ptr(), aw_out.data_ptr(), chol.data_ptr(),
                                                kdev.data_ptr()), what="refresh_basis_async")
        cb = N.CBasis()
        cb.k, cb.d_w, cb.d_aw, cb.d_chol = kmax, w_out.data_ptr(), aw_out.data_ptr(), chol.data_ptr()
        bufs = (w_out, aw_out, chol, kdev, w_src)
    return kmax, cb, kdev, bufs, valid


def prepare_refresh(job, a_next):
    """Enqueue, right behind `job`'s work, the refresh the NEXT solve of the
    sequence will use (its basis is the extraction `job` enqueued): the host
    does this while the device is still busy with `job`'s solve, so the
    refresh's launches never wait for the host.  Hand the result to the next
    solve_next_async(..., prepared=...); unused (the sequence stopped) it is
    simply dropped."""
    op = as_operator(a_next)
    return _PreparedRefresh(job.pending, op, *_enqueue_refresh(job.pending, op, op.n, torch.cuda.current_stream()))


def solve_next_async(state, a, b, ax0=None, ax0_of=None, prepared=None, extract=True, need_aw=True):
    """Enqueue refresh + solve of the next system of a sequence and the
    extraction of the basis after it (device data only, nothing waits).
    Returns (x, job); job.finish() completes the report and the new state.
    ``ax0`` = a @ ax0_of, precomputed by the caller (gpc's fused system
    build), stands in for the warm start's first product when ``ax0_of`` is
    the sequence's last solution.  ``prepared``: the refresh enqueued ahead by
    prepare_refresh (used when it matches this state's basis and operator).
    ``extract=False``: the caller will not solve another system of the
    sequence (gpc's last Newton step), so the next basis is not extracted;
    the returned state then carries no basis.  ``need_aw=False``: the caller
    refreshes the next basis against its next matrix before any use (gpc's
    Newton loop: A changes every step), so the extraction's AW_next for the
    current matrix is not formed (the basis then carries no AW)."""
    op = as_operator(a)
    bd = D.to_dev(b, 1)
    n = bd.shape[0]
    if op.n != n:
        raise DimensionMismatch(f"system shapes {op.shape}, {tuple(bd.shape)}")
    if state.selection not in (SELECT_SMALLEST, SELECT_LARGEST):
        raise ValueError(f"unknown selection {state.selection!r}")
    x_prev = D.zeros(n) if state.x_last is None else D.to_dev(state.x_last, 1)
    t0 = time.perf_counter()
    main = torch.cuda.current_stream()
    pending = object.__getattribute__(state, "basis")
    if ax0 is not None and (ax0_of is None or ax0_of is not state.x_last):
        ax0 = None
    if isinstance(pending, _PendingBasis) and ax0 is None and (prepared is None or prepared.basis_obj is not pending):
        # the warm start's first product A x_prev needs no basis: it runs
        # while the extraction of the basis is still going on
        ax0 = op.matvec_dev(x_prev)
    if prepared is not None and prepared.basis_obj is pending and prepared.op is op:
        kmax, cb, kdev, bufs, valid = prepared.kmax, prepared.cb, prepared.kdev, prepared.bufs, prepared.valid
        if ax0 is None and isinstance(pending, _PendingBasis):
            ax0 = op.matvec_dev(x_prev)
    else:
        # (the pending extraction is joined right before the refresh launch:
        # the host-side set-up of the refresh then overlaps the device's work)
        kmax, cb, kdev, bufs, valid = _enqueue_refresh(pending, op, n, main)
    cfg = state.cfg
    log = KrylovLog(n, cfg.ell, kmax)
    max_iters = 10 * n if cfg.max_iters is None else cfg.max_iters
    sh = D.empty(_STATUS_WORDS + max_iters + 1)   # status words, then the residual history
    status = sh[:_STATUS_WORDS].view(torch.int64)
    hist = sh[_STATUS_WORDS:]
    x = D.empty(n)
    clog = log.c_struct()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    N.check(N.lib().dcg_solve_async(D.ctx(), D.stream(), ctypes.byref(op.c_struct()), bd.data_ptr(),
                                    x_prev.data_ptr(), ctypes.byref(cb) if cb is not None else None,
                                    ctypes.byref(cfg.c_struct()), x.data_ptr(), ctypes.byref(clog),
                                    hist.data_ptr(), kdev.data_ptr() if kdev is not None else None,
                                    status.data_ptr(), ax0.data_ptr() if ax0 is not None else None),
            what="solve_async")
    ev_end = torch.cuda.Event(enable_timing=True)
    ev_end.record()
    nxt = None
    if state.k > 0 and extract:
        # The next basis, extracted straight behind the solve (its sizes come
        # from the solve's status block on the device): the SM-wide column work
        # (Z / AZ, F, G) on the main stream, then the single-CTA pencil and
        # the tail on the side stream, overlapping the caller's next work
        # (the Newton update's K-products leave the pencil an SM of its own).
        k = state.k
        theta = D.empty(k)
        w_next = D.empty(n, k)
        aw_next = D.empty(n, k) if need_aw else None
        result = torch.empty(4, dtype=torch.int64, device=D.device())
        sel = N.DCG_SELECT_LARGEST if state.selection == SELECT_LARGEST else N.DCG_SELECT_SMALLEST
        args = (D.ctx(1), None, n, ctypes.byref(clog), status.data_ptr(), ctypes.byref(cb) if cb is not None else None,
                k, sel, theta.data_ptr(), w_next.data_ptr(), aw_next.data_ptr() if need_aw else None,
                result.data_ptr())
        N.check(N.lib().dcg_ritz_extract_dev(*args[:1], main.cuda_stream, *args[2:], 1), 0, "ritz_extract_dev")
        gathered = torch.cuda.Event()
        gathered.record()
        side = D.side_stream()
        side.wait_event(gathered)
        with torch.cuda.stream(side):
            N.check(N.lib().dcg_ritz_extract_dev(*args[:1], side.cuda_stream, *args[2:], 3), 0, "ritz_extract_dev")
            event = torch.cuda.Event()
            event.record(side)

        def tail(stream, args=args, dev=D.device().index):
            # uscale + wnext: SM-wide, so they run on the joining stream (the
            # main one) rather than in the SMs the side stream is left.  They
            # read stages 1-3's intermediates from the slot-1 workspace; if
            # another extraction was enqueued there since (an interleaved
            # sequence), the whole extraction is re-run from its inputs (the
            # log, the basis used, the solve's status block: kept alive) on
            # the joining stream in the slot-0 workspace, with the same values.
            if _slot1_owner.get(dev) is nxt:
                N.check(N.lib().dcg_ritz_extract_dev(*args[:1], stream.cuda_stream, *args[2:], 4), 0,
                        "ritz_extract_dev")
            else:
                N.check(N.lib().dcg_ritz_extract_dev(D.ctx(0), stream.cuda_stream, *args[2:], 0), 0,
                        "ritz_extract_dev")

        nxt = _PendingBasis(event, result, w_next, aw_next, (log, bufs, theta, status), tail)
        _slot1_owner[D.device().index] = nxt
    job = _AsyncSolve(state, x, log, hist, status, bufs, ev0, ev_end, t0, cfg, nxt, consumed=valid, combined=sh)
    job.hoisted = ax0 is not None   # A x_prev came from outside: the solve kernel skips that product
    return x, job


def harmonic_ritz_extract(log, prev_basis, k, selection=SELECT_SMALLEST):
    """Extract k approximate eigenvectors from a finished solve (recycle.py:95-159).

    Raises BasisDeficient when fewer than k independent columns remain."""
    return _extract_dev(log, prev_basis, int(k), selection)


def solve_next(state, a, b, defer_extraction=False):
    """Solve the next system of a sequence, recycling the deflation basis
    (recycle.py:162-203).  Returns (x, new_state).

    With ``defer_extraction`` the harmonic-Ritz extraction of the next basis
    runs on a side stream and ``new_state.basis`` resolves when first read
    (the next solve), so callers can overlap independent work with it."""
    host = not isinstance(b, torch.Tensor)
    if host:
        b = np.ascontiguousarray(b, dtype=np.float64)
    op = as_operator(a)
    bd = D.to_dev(b, 1)
    n = bd.shape[0]
    if op.n != n:
        raise DimensionMismatch(f"system shapes {op.shape}, {tuple(bd.shape)}")
    x_prev = D.zeros(n) if state.x_last is None else D.to_dev(state.x_last, 1)
    if x_prev.shape[0] != n:
        raise DimensionMismatch(f"system shapes {op.shape}, {tuple(bd.shape)}, {tuple(x_prev.shape)}")

    used = None
    if state.basis is not None and state.basis.k > 0:
        try:
            used = _refresh_dev(op, state.basis.w_dev)
        except BasisDeficient:
            used = None
    t0 = time.perf_counter()
    x, report, log = _solve_dev(op, bd, x_prev, used if (used is not None and used.k > 0) else None, state.cfg, t0)

    nxt = None
    if state.k > 0 and defer_extraction:
        nxt = _extract_async(log, used, state.k, state.selection)
    elif state.k > 0:
        try:
            ext = _extract_dev(log, used, state.k, state.selection)
            if ext.w_next_dev.shape[1] > 0:
                nb = RecycleBasis.__new__(RecycleBasis)
                nb.w_dev, nb.aw_dev, nb.chol_dev = ext.w_next_dev, ext.aw_next_dev, None
                nxt = nb
        except BasisDeficient:
            nxt = None
    x_out = x.cpu().numpy() if host else x
    new_state = replace(state, basis=nxt, x_last=x_out if host else x, history=state.history + [report])
    return x_out, new_state


# ---------------------------------------------------------------------------
# Diagnostics (recycle.py:206-231).  O(n^3) and test/report
# only.  The reference runs its cyclic Jacobi (sym_eigen) on the explicit
# matrices; here n <= DCG_MAX_T runs the same Jacobi kernel on the device and
# larger n the cuSOLVER symmetric eigensolver (eigenvalues equal to rounding).
# The deflated operator P_W A = A - AW (W'AW)^-1 W'A is formed on the device
# with the basis' own Cholesky factor (solvers.py:107-115).
# ---------------------------------------------------------------------------
def _sym_eigvals_dev(m: torch.Tensor) -> np.ndarray:
    n = m.shape[0]
    if n <= N.MAX_T:
        from .linalg import sym_eigen

        return np.asarray(sym_eigen(m).values)
    return torch.linalg.eigvalsh(m).cpu().numpy()


def _explicit(a) -> torch.Tensor:
    if isinstance(a, DenseOperator):
        return a.dense_dev()
    op = as_operator(a)   # validates symmetry (require_symmetric)
    return op.dense_dev()


def condition_numbers(a, k):
    """(kappa, kappa_eff) = (lambda_n / lambda_1, lambda_n / lambda_{k+1}) (recycle.py:206-212)."""
    m = _explicit(a)
    n = m.shape[0]
    if not 0 <= k < n:
        raise ValueError(f"k must be in [0, n), got {k}")
    values = _sym_eigvals_dev(m)
    return float(values[-1] / values[0]), float(values[-1] / values[k])


def deflated_spectrum(a, basis):
    """Eigenvalues (ascending) of the deflated operator P_W A (recycle.py:215-231)."""
    m = _explicit(a)
    if basis is None or basis.k == 0:
        return _sym_eigvals_dev(m)
    low = basis.ensure_factored_dev()
    k = basis.k
    low = low[:k, :k]
    wta = basis.w_dev.T @ m                                  # k x n
    y = torch.linalg.solve_triangular(low, wta, upper=False)
    y = torch.linalg.solve_triangular(low.T, y, upper=True)  # (W'AW)^-1 W'A
    pm = m - basis.aw_dev @ y
    scale = max(float(pm.abs().max()), 1e-300)
    if float((pm - pm.T).abs().max()) <= 1e-8 * scale:
        return _sym_eigvals_dev(0.5 * (pm + pm.T))
    values = torch.linalg.eigvals(pm).real
    return np.sort(values.cpu().numpy())
