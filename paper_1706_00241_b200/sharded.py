"""Row-sharded def-CG over R ranks, one process per GPU.

K is partitioned into contiguous row slabs: rank r owns rows
[r * ceil(n / R), ...) of K and the same rows of x, r, p, Ap (and of W, AW).
With that uniform partition the padded all-gather buffer (R x ceil(n / R))
holds the full vector in its first n entries, so no reordering is needed.

One iteration of the reference's _run_loop (solvers.py:131-204) becomes

    all-gather p                  (8 n / R bytes per rank)
    dcg_shard_apply_dot           local GEMV over the slab + p'Ap partial
    all-reduce(1)
    dcg_shard_update              alpha, x, r, partials [r'r, AW'r]
    all-reduce(1 + k)
    dcg_shard_direction           beta, mu = chol_solve(L, AW'r), p, rel, done

The scalars live in a device-resident dcg_shard_state.  Iterations are
enqueued `poll` at a time and the host reads the done flag once per chunk;
every rank enqueues the same kernels and collectives (kernels after
convergence are no-ops), and the all-reduced values are bit-identical on all
ranks, so all ranks stop together.

The small recycling steps run redundantly on every rank, on all-gathered data
(W, AW are n x k, the Krylov log (2m + 1) x n): refresh_basis's Gram
factorisation with pruning (recycle.py:66-92) and harmonic_ritz_extract
(recycle.py:95-159) use the single-GPU kernels, whose results are
deterministic, so every rank holds the same basis.  Each rank keeps W / AW
whole (n x k) and uses its rows.

The collectives go through a `comm` object (TorchComm: torch.distributed with
NCCL on GPUs; the CPU tests use gloo) and the local arithmetic through a
`backend` (DeviceShardBackend: the C ABI, include/defcg_b200.h L5).  The host
logic here is the same for both.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import BasisDeficient, BreakdownZeroCurvature
from .solvers import SolveReport, SolverConfig, TERM_CONVERGED, TERM_MAX_ITERS

# ---------------------------------------------------------------------------
# partition and communication
# ---------------------------------------------------------------------------


def row_block(n: int, world: int) -> int:
    return max(1, -(-n // world))


def row_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """(row0, rows) of `rank` under the uniform ceil(n / world) partition."""
    mb = row_block(n, world)
    r0 = min(n, rank * mb)
    return r0, max(0, min(n, r0 + mb) - r0)


class SelfComm:
    """world = 1: collectives are identities."""

    rank, world = 0, 1

    def allgather(self, local: torch.Tensor, full: torch.Tensor):
        full[: local.shape[0]].copy_(local)

    def allreduce(self, buf: torch.Tensor):
        return buf


class TorchComm:
    """torch.distributed collectives (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._pad = {}

    def allgather(self, local: torch.Tensor, full: torch.Tensor):
        """`full` holds world x mb entries per leading index (mb = the padded
        block); `local` holds this rank's rows (may be shorter)."""
        mb = full.shape[0] // self.world
        if local.shape[0] == mb:
            src = local
        else:
            key = (mb,) + tuple(local.shape[1:]) + (local.device.type,)
            src = self._pad.get(key)
            if src is None:
                src = torch.zeros((mb,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
                self._pad[key] = src
            src[: local.shape[0]].copy_(local)
        src = src.contiguous()
        try:
            self.dist.all_gather_into_tensor(full, src, group=self.group)
        except (RuntimeError, NotImplementedError):   # backends without the fused form
            parts = list(full.view((self.world,) + tuple(src.shape)).unbind(0))
            self.dist.all_gather(parts, src, group=self.group)

    def allreduce(self, buf: torch.Tensor):
        self.dist.all_reduce(buf, op=self.dist.ReduceOp.SUM, group=self.group)
        return buf


# ---------------------------------------------------------------------------
# operator
# ---------------------------------------------------------------------------


@dataclass
class TileShare:
    """This rank's share of K's packed lower-triangle tiles, [t_lo, t_hi) of
    dcg_shard_tile_range (an equal-cost split of the tile sequence), one
    contiguous device buffer of 32 KB tiles."""

    kp: torch.Tensor
    t_lo: int
    t_hi: int
    rank: int
    world: int


def tile_range(n: int, world: int, rank: int) -> tuple[int, int]:
    lo, hi = ctypes.c_longlong(0), ctypes.c_longlong(0)
    N.check(N.lib().dcg_shard_tile_range(n, rank, world, ctypes.byref(lo), ctypes.byref(hi)), what="tile_range")
    return int(lo.value), int(hi.value)


class ShardedOperator:
    """This rank's slab of A = shift I + S K S: rows [row0, row0 + rows) of K
    (device, leading dimension ldk), the full scale vector s (n) or None.

    With a ``share`` (TileShare) the solve's products read the rank's packed
    tile share instead (half the slab's bytes) and the solve runs on
    replicated vectors with one all-reduce of n doubles per product; the slab
    still serves the once-per-system products (refresh, Newton glue)."""

    def __init__(self, kslab: torch.Tensor, n: int, ldk: int, row0: int, rows: int, s=None, shift: float = 0.0,
                 share: TileShare | None = None):
        self.kslab, self.n, self.ldk, self.row0, self.rows = kslab, int(n), int(ldk), int(row0), int(rows)
        self.s = s
        self.shift = float(shift)
        self.share = share

    def scaled(self, s, shift: float) -> "ShardedOperator":
        return ShardedOperator(self.kslab, self.n, self.ldk, self.row0, self.rows, s, shift, self.share)

    def share_struct(self) -> N.COperator:
        """The tile share as a DENSE_SYM operator over all n rows."""
        c = N.COperator()
        c.kind = N.DCG_OP_DENSE_SYM
        c.n = self.n
        c.row0 = 0
        c.rows = self.n
        c.d_kp = self.share.kp.data_ptr() if self.share.kp.numel() else None
        c.ldk = self.n + (self.n & 1)
        c.d_s = self.s.data_ptr() if self.s is not None else None
        c.shift = self.shift
        return c

    def c_struct(self) -> N.COperator:
        c = N.COperator()
        c.kind = N.DCG_OP_DENSE
        c.n = self.n
        c.row0 = self.row0
        c.rows = self.rows
        c.d_k = self.kslab.data_ptr()
        c.ldk = self.ldk
        c.d_s = self.s.data_ptr() if self.s is not None else None
        c.shift = self.shift
        return c


class ShardedRbfOperator:
    """This rank's slab of the matrix-free A = shift I + S K S (config 5):
    rows [row0, row0 + rows) of the RBF kernel, regenerated from the
    replicated points X on every product (the row-owned tensor-pipe kernel,
    csrc/rbfmma.cuh); nothing of size n^2 / R is stored."""

    def __init__(self, x: torch.Tensor, var: float, inv_two_ell2: float, diag: float, row0: int, rows: int, s=None,
                 shift: float = 0.0, rank: int = 0, world: int = 1, symmetric: bool = True):
        self.x = x
        self.n, self.row0, self.rows = int(x.shape[0]), int(row0), int(rows)
        self.var, self.inv_two_ell2, self.diag = float(var), float(inv_two_ell2), float(diag)
        self.s = s
        self.shift = float(shift)
        # symmetric: the solve's products evaluate this rank's share of the
        # lower-triangle tiles and all-reduce an n-vector (half the pairs of
        # the row slab); otherwise the row slab is evaluated in full
        self.rank, self.world, self.symmetric = int(rank), int(world), bool(symmetric)

    def scaled(self, s, shift: float) -> "ShardedRbfOperator":
        return ShardedRbfOperator(self.x, self.var, self.inv_two_ell2, self.diag, self.row0, self.rows, s, shift,
                                  self.rank, self.world, self.symmetric)

    def c_struct(self) -> N.COperator:
        c = N.COperator()
        c.kind = N.DCG_OP_RBF
        c.n = self.n
        c.row0 = self.row0
        c.rows = self.rows
        c.d_k = None
        c.ldk = 0
        c.d_x = self.x.data_ptr() if self.n else None
        c.dim = int(self.x.shape[1])
        c.var = self.var
        c.inv_two_ell2 = self.inv_two_ell2
        c.diag = self.diag
        c.d_s = self.s.data_ptr() if self.s is not None else None
        c.shift = self.shift
        return c


def sharded_rbf_kernel(x, params, jitter=None, comm=None, matrix_free=False, tile_share=True):
    """This rank's rows of the RBF Gram (gpc.py:82-98), built on device from
    the replicated data X (n x d, a few MB) - Gram blocks never cross PCIe.
    With ``matrix_free`` the slab is never stored: a ShardedRbfOperator
    regenerates it on every product (config 5).  With ``tile_share`` the rank
    also builds its share of the packed lower-triangle tiles (entries bitwise
    the slab's), which the solves stream instead of the slab."""
    comm = comm or SelfComm()
    xd = D.to_dev(x, 2)
    n, dim = xd.shape
    var = params.signal_sd**2
    jitter = 1e-8 * var if jitter is None else float(jitter)
    if jitter < 0.0:
        raise ValueError("jitter must be non-negative")
    r0, rows = row_range(n, comm.world, comm.rank)
    if matrix_free:
        return ShardedRbfOperator(xd.contiguous(), var, 1.0 / (2.0 * params.lengthscale**2), var + jitter, r0, rows,
                                  rank=comm.rank, world=comm.world)
    ld = D.padded_ld(n)
    kslab = D.zeros(max(rows, 1), ld)
    if rows:
        N.check(N.lib().dcg_k_rbf_gram(D.ctx(), D.stream(), xd.data_ptr(), n, dim, var,
                                       1.0 / (2.0 * params.lengthscale**2), jitter, kslab.data_ptr(), ld, r0, rows),
                what="rbf_gram")
    share = None
    if tile_share and n:
        t_lo, t_hi = tile_range(n, comm.world, comm.rank)
        kp = D.empty(max(t_hi - t_lo, 0) * 4096)
        if t_hi > t_lo:
            N.check(N.lib().dcg_k_rbf_gram_packed(D.ctx(), D.stream(), xd.data_ptr(), n, dim, var,
                                                  1.0 / (2.0 * params.lengthscale**2), jitter, t_lo, t_hi,
                                                  kp.data_ptr()), what="rbf_gram_packed")
        share = TileShare(kp, t_lo, t_hi, comm.rank, comm.world)
    return ShardedOperator(kslab, n, ld, r0, rows, share=share)


# ---------------------------------------------------------------------------
# device backend (the C ABI)
# ---------------------------------------------------------------------------


def _p(t):
    return None if t is None else t.data_ptr()


class DeviceShardBackend:
    """Local arithmetic of one rank through the L5 entry points."""

    def __init__(self, slot: int = 0):
        self.slot = slot

    def ctx(self):
        return D.ctx(self.slot)

    def stream(self):
        return D.stream()

    def empty(self, *shape):
        return D.empty(*shape)

    def zeros(self, *shape):
        return D.zeros(*shape)

    def new_state(self):
        return D.zeros(N.SHARD_STATE_DOUBLES)

    def read_state(self, st: torch.Tensor) -> dict:
        h = st.cpu()
        i = h.view(torch.int64)
        return {"rr": float(h[N.SHARD_RR]), "norm_b": float(h[N.SHARD_NORM_B]), "rel": float(h[N.SHARD_REL]),
                "it": int(i[N.SHARD_IT]), "done": int(i[N.SHARD_DONE]), "status": int(i[N.SHARD_STATUS]),
                "info": int(i[N.SHARD_INFO])}

    def residual(self, op, vfull, b, r, state=None):
        cop = op.c_struct()
        N.check(N.lib().dcg_shard_residual(self.ctx(), self.stream(), ctypes.byref(cop), _p(vfull), _p(b), _p(r),
                                           _p(state)), what="shard_residual")

    def apply_dot(self, op, vfull, out, part, state):
        cop = op.c_struct()
        N.check(N.lib().dcg_shard_apply_dot(self.ctx(), self.stream(), ctypes.byref(cop), _p(vfull), _p(out),
                                            _p(part), _p(state)), what="shard_apply_dot")

    def sym_partial(self, op, vfull, t, state=None):
        cop = op.c_struct()
        N.check(N.lib().dcg_shard_rbf_sym_partial(self.ctx(), self.stream(), ctypes.byref(cop), op.rank, op.world,
                                                  _p(vfull), _p(t), _p(state)), what="shard_rbf_sym_partial")

    def tiles_partial(self, op, vfull, t, state=None):
        cop = op.share_struct()
        N.check(N.lib().dcg_shard_tiles_partial(self.ctx(), self.stream(), ctypes.byref(cop), op.share.rank,
                                                op.share.world, _p(vfull), _p(t), _p(state)),
                what="shard_tiles_partial")

    def epilogue(self, mode, op, vfull, b, t, out, part, state=None):
        cop = op.share_struct() if getattr(op, "share", None) is not None else op.c_struct()
        N.check(N.lib().dcg_shard_epilogue(self.ctx(), self.stream(), mode, ctypes.byref(cop), _p(vfull), _p(b), _p(t),
                                           _p(out), _p(part), _p(state)), what="shard_epilogue")

    def partials(self, rows, k, u, w, m, part):
        N.check(N.lib().dcg_shard_partials(self.ctx(), self.stream(), rows, k, _p(u), _p(w), _p(m), _p(part)),
                what="shard_partials")

    def start(self, rows, k, red, chol, w, xprev, x0, state, tol, max_iters, ell):
        N.check(N.lib().dcg_shard_start(self.ctx(), self.stream(), rows, k, _p(red), _p(chol), _p(w), _p(xprev),
                                        _p(x0), _p(state), tol, max_iters, ell), what="shard_start")

    def start_r(self, rows, k, red, chol, w, aw, xprev, x0, r, state, tol, max_iters, ell):
        N.check(N.lib().dcg_shard_start_r(self.ctx(), self.stream(), rows, k, _p(red), _p(chol), _p(w), _p(aw),
                                          _p(xprev), _p(x0), _p(r), _p(state), tol, max_iters, ell),
                what="shard_start_r")

    def begin(self, rows, k, red, chol, w, r, p, x, state, hist, log):
        N.check(N.lib().dcg_shard_begin(self.ctx(), self.stream(), rows, k, _p(red), _p(chol), _p(w), _p(r), _p(p),
                                        _p(x), _p(state), _p(hist), _p(log.r), _p(log.p), _p(log.mu)),
                what="shard_begin")

    def update(self, mode, rows, k, red_d, x, r, p, ap, aw, part, state, log):
        N.check(N.lib().dcg_shard_update(self.ctx(), self.stream(), mode, rows, k, _p(red_d), _p(x), _p(r), _p(p),
                                         _p(ap), _p(aw), _p(part), _p(state), _p(log.r), _p(log.d), _p(log.alpha),
                                         _p(log.beta)), what="shard_update")

    def step(self, op, rows, k, t, x, r, p, ap, w, aw, chol, state, hist, log):
        """epilogue(0) + update(0) + direction on replicated vectors in one cooperative launch."""
        N.check(N.lib().dcg_shard_step(self.ctx(), self.stream(), rows, k, _p(t), _p(op.s), float(op.shift), _p(x),
                                       _p(r), _p(p), _p(ap), _p(w), _p(aw), _p(chol), _p(state), _p(hist), _p(log.r),
                                       _p(log.p), _p(log.d), _p(log.alpha), _p(log.beta), _p(log.mu)),
                what="shard_step")

    def direction(self, rows, k, red, chol, w, r, p, state, hist, log):
        N.check(N.lib().dcg_shard_direction(self.ctx(), self.stream(), rows, k, _p(red), _p(chol), _p(w), _p(r),
                                            _p(p), _p(state), _p(hist), _p(log.p), _p(log.mu), _p(log.beta)),
                what="shard_direction")


# ---------------------------------------------------------------------------
# solve
# ---------------------------------------------------------------------------


@dataclass
class ShardLog:
    """This rank's rows of the KrylovLog (solvers.py:54-72): p (ell x rows),
    r ((ell + 1) x rows), d / alpha / beta (ell), mu (ell x k)."""

    p: torch.Tensor
    r: torch.Tensor
    d: torch.Tensor
    alpha: torch.Tensor
    beta: torch.Tensor
    mu: torch.Tensor | None
    m: int = 0
    replicated: bool = False   # rows = n on every rank (tile-share solves)


@dataclass
class ShardBasis:
    """RecycleBasis replicated on every rank: W, AW (n x k) and L (k x k)."""

    w: torch.Tensor
    aw: torch.Tensor
    chol: torch.Tensor

    @property
    def k(self) -> int:
        return int(self.w.shape[1])


def _alloc_log(be, rows, ell, k):
    cap = max(ell, 1)
    return ShardLog(p=be.empty(cap, max(rows, 1)), r=be.empty(cap + 1, max(rows, 1)), d=be.empty(cap),
                    alpha=be.empty(cap), beta=be.empty(cap), mu=be.empty(cap, max(k, 1)) if k else None)


def sharded_solve(op: ShardedOperator, b_loc, x_prev_loc, basis: ShardBasis | None, cfg: SolverConfig | None = None,
                  comm=None, backend=None, poll: int | None = None, ax0=None):
    """CG (basis None or k = 0, solvers.py:207-219) or deflated CG with the
    warm-start correction (solvers.py:222-239) on this rank's rows.  Returns
    (x_loc, SolveReport, ShardLog); every rank gets the same report."""
    cfg = cfg or SolverConfig()
    comm = comm or SelfComm()
    be = backend or DeviceShardBackend()
    if poll is None:
        poll = int(os.environ.get("DCG_SHARD_POLL", "4"))
    t0 = time.perf_counter()
    n, rows, r0 = op.n, op.rows, op.row0
    k = basis.k if basis is not None else 0
    # Tile-share operators: every rank holds the whole vectors and runs the
    # vector phases redundantly (identically: the reductions see the same
    # all-reduced data in the same order); the only exchange is the
    # all-reduce of each product's partial K (s (.) v).
    share = getattr(op, "share", None)
    pcomm = comm
    if share is not None:
        slab_rows, slab_r0 = rows, r0
        if comm.world > 1:
            b_loc = _allgather_vec(comm, be, b_loc[:rows], n).contiguous()
            x_prev_loc = _allgather_vec(comm, be, x_prev_loc[:rows], n).contiguous()
        comm = SelfComm()
        rows, r0 = n, 0
    mb = row_block(n, comm.world)
    ell = int(cfg.ell)
    max_iters = 10 * n if cfg.max_iters is None else int(cfg.max_iters)
    every = int(cfg.recompute_residual_every or 0)

    w_loc = basis.w[r0:r0 + rows] if k else None
    aw_loc = basis.aw[r0:r0 + rows] if k else None
    chol = basis.chol if k else None
    full = be.empty(comm.world * mb)
    x = be.empty(max(rows, 1))
    r = be.empty(max(rows, 1))
    p = be.empty(max(rows, 1))
    ap = be.empty(max(rows, 1))
    part1 = be.zeros(2)
    part2 = be.zeros(2 + k)
    state = be.new_state()
    hist = be.zeros(max_iters + 1)
    log = _alloc_log(be, rows, ell, k)

    # products: the row slab, or this rank's share of the lower-triangle tiles
    # (stored: the tile share; matrix-free: regenerated) + an all-reduce of
    # K (s (.) v)
    sym = getattr(op, "symmetric", False) or share is not None
    tfull = be.empty(max(n, comm.world * mb)) if sym else None

    def partial(st):
        if share is not None:
            be.tiles_partial(op, full, tfull, st)
        else:
            be.sym_partial(op, full, tfull, st)
        pcomm.allreduce(tfull[:n] if share is not None else tfull)

    def residual(bvec, out, st=None):
        if sym:
            partial(st)
            be.epilogue(1, op, full, bvec, tfull, out, None, st)
        else:
            be.residual(op, full, bvec, out, st)

    def apply_dot(out, part, st):
        if sym:
            partial(st)
            be.epilogue(0, op, full, None, tfull, out, part, st)
        else:
            be.apply_dot(op, full, out, part, st)

    # ---- prologue: norm_b, warm start, r_0, mu_0, p_0 ----------------------
    # ax0 (tile shares: all n rows): A x_prev computed by the caller together
    # with the Newton system's product, which saves this solve's first product
    use_ax0 = ax0 is not None and share is not None
    if k:
        if use_ax0:
            torch.sub(b_loc[:n], ax0[:n], out=r[:n])         # r_prev = b - A x_prev
        else:
            comm.allgather(x_prev_loc, full)
            residual(b_loc, r)                             # r_prev = b - A x_prev
        be.partials(rows, k, b_loc, r, w_loc, part2)       # [b'b, W' r_prev]
        comm.allreduce(part2)
        # x_0 = x_prev + W c and r_0 = r_prev - (AW) c: no second product
        be.start_r(rows, k, part2, chol, w_loc, aw_loc, x_prev_loc, x, r, state, float(cfg.tol), max_iters, ell)
    else:
        be.partials(rows, 0, b_loc, None, None, part2)     # [b'b]
        comm.allreduce(part2)
        be.start(rows, k, part2, chol, w_loc, x_prev_loc, x, state, float(cfg.tol), max_iters, ell)
        if use_ax0:
            torch.sub(b_loc[:n], ax0[:n], out=r[:n])         # r_0 = b - A x_0, x_0 = x_prev
        else:
            comm.allgather(x[:rows], full)
            residual(b_loc, r)                             # r_0 = b - A x_0
    be.partials(rows, k, r, r, aw_loc, part2)              # [r0'r0, AW' r0]
    comm.allreduce(part2)
    be.begin(rows, k, part2, chol, w_loc, r, p, x, state, hist, log)

    # ---- iterations, `poll` per host check -----------------------------------
    fused = share is not None and hasattr(be, "step") and not os.environ.get("DCG_SHARD_NO_FUSED_STEP")
    j = 0
    while True:
        st = be.read_state(state)
        if st["done"]:
            break
        for _ in range(max(1, poll)):
            j += 1
            if fused and not (every > 0 and j % every == 0):
                # tile shares: the vectors are replicated, so the iteration is
                # the share's product, its all-reduce and ONE launch for the rest
                be.tiles_partial(op, p, tfull, state)   # (p holds all n rows: no gather copy)
                pcomm.allreduce(tfull[:n])
                be.step(op, rows, k, tfull, x, r, p, ap, w_loc, aw_loc, chol, state, hist, log)
                continue
            comm.allgather(p[:rows], full)
            apply_dot(ap, part1, state)
            comm.allreduce(part1)
            if every > 0 and j % every == 0:               # true residual (solvers.py:175-177)
                be.update(1, rows, k, part1, x, r, p, ap, aw_loc, part2, state, log)
                comm.allgather(x[:rows], full)
                residual(b_loc, r, state)
                be.update(2, rows, k, None, x, r, p, ap, aw_loc, part2, state, log)
            else:
                be.update(0, rows, k, part1, x, r, p, ap, aw_loc, part2, state, log)
            comm.allreduce(part2)
            be.direction(rows, k, part2, chol, w_loc, r, p, state, hist, log)

    if st["status"] == N.DCG_E_BREAKDOWN:
        raise BreakdownZeroCurvature(st["info"])
    its = st["it"]
    log.m = min(its, ell)
    history = hist[: its + 1].cpu().tolist()
    conv = st["rel"] <= cfg.tol
    rep = SolveReport(its, history, conv, time.perf_counter() - t0, TERM_CONVERGED if conv else TERM_MAX_ITERS)
    if share is not None:
        log.replicated = True   # all n rows on every rank
        return x[slab_r0:slab_r0 + slab_rows], rep, log
    return x[:rows], rep, log


# ---------------------------------------------------------------------------
# recycling on gathered data
# ---------------------------------------------------------------------------


def _gather_rows(comm, be, local: torch.Tensor, n: int) -> torch.Tensor:
    """(rows x c) local row block -> (n x c) on every rank."""
    mb = row_block(n, comm.world)
    c = local.shape[1] if local.dim() == 2 else 1
    full = be.empty(comm.world * mb, c) if local.dim() == 2 else be.empty(comm.world * mb)
    comm.allgather(local, full)
    return full[:n]


def _gather_log(comm, be, log: ShardLog, n: int, rows: int):
    """Full (n-row) KrylovLog buffers of the first m logged iterations."""
    from .solvers import KrylovLog

    m = log.m
    cap = log.p.shape[0]
    full = KrylovLog(n, cap, log.mu.shape[1] if log.mu is not None else 0)
    mb = row_block(n, comm.world)
    # gather (vectors x rows) blocks as rows x vectors so the row-block gather applies
    pr = torch.cat([log.p[:m, :rows], log.r[: m + 1, :rows]], dim=0).t().contiguous()
    g = be.empty(comm.world * mb, pr.shape[1])
    comm.allgather(pr, g)
    g = g[:n].t()
    if m:
        full._p[:m].copy_(g[:m])
    full._r[: m + 1].copy_(g[m:])
    full._s[0, :m].copy_(log.d[:m])
    full._s[1, :m].copy_(log.alpha[:m])
    full._s[2, :m].copy_(log.beta[:m])
    if log.mu is not None and m:
        full._mu[:m].copy_(log.mu[:m])
    full.m = m
    return full


def sharded_refresh_basis(op: ShardedOperator, w_full: torch.Tensor, comm=None, backend=None) -> ShardBasis:
    """refresh_basis (recycle.py:80-92) for the sharded operator: AW's rows by
    the local slab product, all-gathered; W'AW factored with failing-pivot
    pruning redundantly (and identically) on every rank."""
    comm = comm or SelfComm()
    be = backend or DeviceShardBackend()
    n, k = w_full.shape
    if k == 0:
        return ShardBasis(w_full, w_full.clone(), be.empty(0, 0))
    rows = op.rows
    share = getattr(op, "share", None)
    if share is not None and share.world == 1 and N.lib().dcg_block_uses_packed(k):
        # one rank holds every tile: the symmetric block product over the
        # packed share (half the slab's bytes) gives all n rows of AW at once
        aw = be.empty(n, k)
        cop = op.share_struct()
        N.check(N.lib().dcg_op_apply_block(be.ctx(), be.stream(), ctypes.byref(cop), w_full.contiguous().data_ptr(), k,
                                           aw.data_ptr()), what="refresh_basis")
    else:
        aw_loc = be.empty(max(rows, 1), k)
        cop = op.c_struct()
        if rows:
            N.check(N.lib().dcg_op_apply_block(be.ctx(), be.stream(), ctypes.byref(cop), w_full.data_ptr(), k,
                                               aw_loc.data_ptr()), what="refresh_basis")
        aw = _gather_rows(comm, be, aw_loc[:rows], n).contiguous()
    w = w_full.contiguous().clone()
    chol = be.empty(k, k)
    kout, info = ctypes.c_longlong(k), ctypes.c_longlong(0)
    rc = N.lib().dcg_gram_factor(be.ctx(), be.stream(), w.data_ptr(), aw.data_ptr(), n, k, 1, chol.data_ptr(),
                                 ctypes.byref(kout), ctypes.byref(info))
    N.check(rc, info.value, "refresh_basis")
    kk = int(kout.value)
    return ShardBasis(w.view(-1)[: n * kk].view(n, kk), aw.view(-1)[: n * kk].view(n, kk),
                      chol.view(-1)[: kk * kk].view(kk, kk))


def sharded_extract(log: ShardLog, prev: ShardBasis | None, k: int, selection: str, n: int, rows: int, comm=None,
                    backend=None) -> ShardBasis | None:
    """harmonic_ritz_extract (recycle.py:95-159) on the gathered log, run
    redundantly on every rank; returns W_next / AW_next (n x k, factor
    computed at the next refresh) or raises BasisDeficient."""
    from .recycle import RecycleBasis, _extract_dev

    comm = comm or SelfComm()
    be = backend or DeviceShardBackend()
    flog = _gather_log(SelfComm(), be, log, n, n) if log.replicated else _gather_log(comm, be, log, n, rows)
    pb = None
    if prev is not None and prev.k:
        pb = RecycleBasis.__new__(RecycleBasis)
        pb.w_dev, pb.aw_dev, pb.chol_dev = prev.w, prev.aw, prev.chol
    ext = _extract_dev(flog, pb, int(k), selection)
    # the device tensors (the RitzExtraction's numpy properties copy to the host)
    if ext.w_next_dev.shape[1] == 0:
        return None
    return ShardBasis(ext.w_next_dev.contiguous(), ext.aw_next_dev.contiguous(), be.empty(0, 0))


@dataclass
class ShardSequenceState:
    """SequenceState (recycle.py:49-63) for the sharded solver: the basis is
    replicated (n x k), x_last holds this rank's rows."""

    k: int
    cfg: SolverConfig = field(default_factory=SolverConfig)
    selection: str = "smallest"
    basis: ShardBasis | None = None
    x_last: torch.Tensor | None = None
    history: list = field(default_factory=list)


def sharded_solve_next(state: ShardSequenceState, op: ShardedOperator, b_loc, comm=None, backend=None, ax0=None):
    """solve_next (recycle.py:162-203) on row shards: refresh (BasisDeficient
    -> plain CG), solve, extraction (BasisDeficient -> no basis)."""
    comm = comm or SelfComm()
    be = backend or DeviceShardBackend()
    rows = op.rows
    x_prev = state.x_last if state.x_last is not None else be.zeros(max(rows, 1))
    used = None
    if state.basis is not None and state.basis.k > 0:
        try:
            used = sharded_refresh_basis(op, state.basis.w, comm, be)
        except BasisDeficient:
            used = None
    x, rep, log = sharded_solve(op, b_loc, x_prev[:rows], used, state.cfg, comm, be, ax0=ax0)
    nxt = None
    if state.k > 0:
        try:
            nxt = sharded_extract(log, used, state.k, state.selection, op.n, rows, comm, be)
        except BasisDeficient:
            nxt = None
    return x, replace(state, basis=nxt, x_last=x, history=state.history + [rep])


# ---------------------------------------------------------------------------
# GPC Laplace-Newton on row shards
# ---------------------------------------------------------------------------


def _share_kv(op: ShardedOperator, v: torch.Tensor, comm, be) -> torch.Tensor:
    """K v (all n rows, on every rank) from the tile shares: each rank's
    partial, then one all-reduce."""
    t = be.empty(op.n)
    be.tiles_partial(op.scaled(None, 0.0), v.contiguous(), t)
    comm.allreduce(t)
    return t


def _allgather_vec(comm, be, local: torch.Tensor, n: int) -> torch.Tensor:
    mb = row_block(n, comm.world)
    full = be.empty(comm.world * mb)
    comm.allgather(local, full)
    return full[:n]


def sharded_laplace_newton(x, y, params=None, cfg: SolverConfig | None = None, newton_tol=1.0, max_newton=30, k=8,
                           selection="largest", comm=None, backend=None, jitter=None, matrix_free=False):
    """laplace_newton(rbf_kernel(x, params), y, "defcg", ...) (gpc.py:212-291)
    with K row-sharded over the ranks of `comm`: every rank builds its slab
    from the replicated X, the n-vectors of the Newton glue (f, a, s, H f + g)
    are replicated (O(n) work, computed identically on every rank), and each
    system is solved by sharded_solve_next.  Returns the list of
    NewtonRecord (f as numpy) - identical on every rank."""
    from .errors import NoProgress
    from .gpc import NewtonRecord

    cfg = cfg or SolverConfig()
    comm = comm or SelfComm()
    be = backend or DeviceShardBackend()
    # `x` is the data matrix (the slab is built here) or a prebuilt kernel slab
    op = x if isinstance(x, (ShardedOperator, ShardedRbfOperator)) else sharded_rbf_kernel(x, params, jitter, comm,
                                                                                             matrix_free)
    kop = op.c_struct()   # the kernel matrix itself (no scaling, no shift)
    n, rows = op.n, op.rows
    yd = D.to_dev(y, 1)
    f = be.zeros(n)
    a = be.zeros(n)
    grad, h = be.empty(n), be.empty(n)
    ll = ctypes.c_double(0.0)
    N.check(N.lib().dcg_gpc_derivs(be.ctx(), be.stream(), n, f.data_ptr(), yd.data_ptr(), grad.data_ptr(),
                                   h.data_ptr(), ctypes.byref(ll)), what="derivs")
    psi_prev = float(ll.value)
    state = ShardSequenceState(k=k, cfg=cfg, selection=selection)
    records = []
    share = getattr(op, "share", None)
    r0 = op.row0
    x_last = None   # the previous solution (all rows), the next solve's warm start
    for it in range(1, max_newton + 1):
        s, inner, b_loc = be.empty(n), be.empty(n), be.empty(max(rows, 1))
        ax0 = None
        if share is not None:
            # gpc.py:175-183 with the product from the tile shares: s = sqrt(h),
            # inner = h f + grad, b = s (.) (K inner), element-wise as the
            # reference rounds them (one rounding per operation); from the
            # second step on the same share pass also gives A x_prev =
            # x_prev + s (.) K (s (.) x_prev), the solve's first product
            torch.sqrt(h, out=s)
            torch.add(torch.mul(h, f), grad, out=inner)
            if x_last is None:
                b_loc[:rows] = torch.mul(s, _share_kv(op, inner, comm, be))[r0:r0 + rows]
            else:
                t = be.empty(2 * n)
                xs = torch.mul(s, x_last)
                cop = op.scaled(None, 0.0).share_struct()
                N.check(N.lib().dcg_shard_tiles_partial2(be.ctx(), be.stream(), ctypes.byref(cop), share.rank,
                                                         share.world, inner.data_ptr(), xs.data_ptr(),
                                                         t.data_ptr(), t[n:].data_ptr()), what="shard_tiles_partial2")
                comm.allreduce(t)
                b_loc[:rows] = torch.mul(s, t[:n])[r0:r0 + rows]
                ax0 = torch.add(x_last, torch.mul(s, t[n:]))
        else:
            N.check(N.lib().dcg_gpc_newton_system(be.ctx(), be.stream(), ctypes.byref(kop), f.data_ptr(),
                                                  grad.data_ptr(), h.data_ptr(), s.data_ptr(), inner.data_ptr(),
                                                  b_loc.data_ptr()), what="newton_system")
        t0 = time.perf_counter()
        x_loc, state = sharded_solve_next(state, op.scaled(s, 1.0), b_loc[:rows], comm, be, ax0=ax0)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        rep = state.history[-1]
        x_full = _allgather_vec(comm, be, x_loc, n).contiguous()
        x_last = x_full
        if share is not None:
            # gpc.py:186-191: a = inner - s (.) x, f = K a (tile shares)
            a = torch.sub(inner, torch.mul(s, x_full))
            f = _share_kv(op, a, comm, be)
        else:
            f_loc = be.empty(max(rows, 1))
            a = be.empty(n)
            N.check(N.lib().dcg_gpc_newton_update(be.ctx(), be.stream(), ctypes.byref(kop), inner.data_ptr(),
                                                  s.data_ptr(), x_full.data_ptr(), yd.data_ptr(), a.data_ptr(),
                                                  f_loc.data_ptr(), grad.data_ptr(), h.data_ptr(), None, None),
                    what="newton_update")
            f = _allgather_vec(comm, be, f_loc[:rows], n).contiguous()
        ll, psi = ctypes.c_double(0.0), ctypes.c_double(0.0)
        N.check(N.lib().dcg_gpc_objective(be.ctx(), be.stream(), n, f.data_ptr(), yd.data_ptr(), a.data_ptr(),
                                          grad.data_ptr(), h.data_ptr(), ctypes.byref(ll), ctypes.byref(psi)),
                what="objective")
        psi = float(psi.value)
        records.append(NewtonRecord(newton_iter=it, psi=psi, loglik=float(ll.value),
                                    solver_iterations=rep.iterations, rel_residual=rep.residual_history[-1],
                                    solve_time_s=dt, residual_history=list(rep.residual_history), f=f.clone()))
        if psi < psi_prev - 1e-6:
            raise NoProgress(f"objective fell from {psi_prev:.9g} to {psi:.9g} at iteration {it}")
        if psi - psi_prev < newton_tol:
            break
        psi_prev = psi
    for r in records:
        r.f = r.f.cpu().numpy()
    return records
