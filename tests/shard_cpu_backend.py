"""CPU restatement of the L5 shard kernels (csrc/shard.cu) for the host-logic
tests of the sharded solver (torch float64 on the CPU; test infrastructure,
never used by the package).  Same state layout and no-op-after-done rules."""

import torch

from paper_1706_00241_b200 import _native as N

F64 = torch.float64


def _chol_solve(L, c):
    y = torch.linalg.solve_triangular(L, c.reshape(-1, 1), upper=False)
    return torch.linalg.solve_triangular(L.t(), y, upper=True).reshape(-1)


class CpuShardBackend:
    def empty(self, *shape):
        return torch.zeros(shape, dtype=F64)

    zeros = empty

    def new_state(self):
        return torch.zeros(N.SHARD_STATE_DOUBLES, dtype=F64)

    @staticmethod
    def _i(st):
        return st.view(torch.int64)

    def read_state(self, st):
        i = self._i(st)
        return {"rr": float(st[N.SHARD_RR]), "norm_b": float(st[N.SHARD_NORM_B]), "rel": float(st[N.SHARD_REL]),
                "it": int(i[N.SHARD_IT]), "done": int(i[N.SHARD_DONE]), "status": int(i[N.SHARD_STATUS]),
                "info": int(i[N.SHARD_INFO])}

    def _done(self, st):
        return st is not None and int(self._i(st)[N.SHARD_DONE]) != 0

    @staticmethod
    def _apply(op, vfull):
        n, r0, rows = op.n, op.row0, op.rows
        v = vfull[:n]
        sv = op.s * v if op.s is not None else v
        t = op.kslab[:rows, :n] @ sv
        if op.s is not None:
            t = op.s[r0:r0 + rows] * t
        return op.shift * v[r0:r0 + rows] + t

    def residual(self, op, vfull, b, r, state=None):
        if self._done(state):
            return
        r[: op.rows] = b[: op.rows] - self._apply(op, vfull)

    def apply_dot(self, op, vfull, out, part, state):
        if self._done(state):
            return
        out[: op.rows] = self._apply(op, vfull)
        part[0] = torch.dot(vfull[op.row0:op.row0 + op.rows], out[: op.rows])

    def partials(self, rows, k, u, w, m, part):
        part[0] = torch.dot(u[:rows], u[:rows])
        if k:
            part[1:1 + k] = m[:rows].t() @ w[:rows]

    def start(self, rows, k, red, chol, w, xprev, x0, state, tol, max_iters, ell):
        x0[:rows] = xprev[:rows] + (w[:rows] @ _chol_solve(chol, red[1:1 + k]) if k else 0.0)
        state.zero_()
        i = self._i(state)
        state[N.SHARD_NORM_B] = float(red[0]) ** 0.5
        state[N.SHARD_TOL] = tol
        i[N.SHARD_MAX_ITERS] = max_iters
        i[N.SHARD_ELL] = ell

    def start_r(self, rows, k, red, chol, w, aw, xprev, x0, r, state, tol, max_iters, ell):
        c = _chol_solve(chol, red[1:1 + k])
        self.start(rows, k, red, chol, w, xprev, x0, state, tol, max_iters, ell)
        r[:rows] = r[:rows] - aw[:rows] @ c

    def begin(self, rows, k, red, chol, w, r, p, x, state, hist, log):
        i = self._i(state)
        nb, tol, ell, mx = float(state[N.SHARD_NORM_B]), float(state[N.SHARD_TOL]), int(i[N.SHARD_ELL]), int(i[N.SHARD_MAX_ITERS])
        rr = float(red[0])
        if nb == 0.0:
            x[:rows] = 0.0
            log.r[0, :rows] = 0.0
            state[N.SHARD_RR], state[N.SHARD_REL] = rr, 0.0
            i[N.SHARD_DONE] = 1
            hist[0] = 0.0
            return
        rel = rr ** 0.5 / nb
        cont = rel > tol and 0 < mx
        mu = _chol_solve(chol, red[1:1 + k]) if k else None
        p[:rows] = r[:rows] - (w[:rows] @ mu if k else 0.0)
        log.r[0, :rows] = r[:rows]
        if cont and ell > 0:
            log.p[0, :rows] = p[:rows]
            if k:
                log.mu[0, :k] = mu
        state[N.SHARD_RR], state[N.SHARD_REL] = rr, rel
        i[N.SHARD_DONE] = 0 if cont else 1
        hist[0] = rel

    def update(self, mode, rows, k, red_d, x, r, p, ap, aw, part, state, log):
        if self._done(state):
            return
        i = self._i(state)
        it, ell = int(i[N.SHARD_IT]), int(i[N.SHARD_ELL])
        if mode != 2:
            d = float(red_d[0])
            if d <= 0.0:
                i[N.SHARD_STATUS], i[N.SHARD_INFO], i[N.SHARD_DONE] = N.DCG_E_BREAKDOWN, it, 1
                return
            alpha = float(state[N.SHARD_RR]) / d
            x[:rows] += alpha * p[:rows]
            if mode == 0:
                r[:rows] -= alpha * ap[:rows]
            state[N.SHARD_ALPHA], state[N.SHARD_D] = alpha, d
            i[N.SHARD_IT] = it + 1
            if it < ell:
                log.d[it], log.alpha[it] = d, alpha
            if mode == 1:
                return
            it += 1
        if it - 1 < ell:
            log.r[it, :rows] = r[:rows]
        self.partials(rows, k, r, r, aw, part)

    def direction(self, rows, k, red, chol, w, r, p, state, hist, log):
        if self._done(state):
            return
        i = self._i(state)
        it, ell, mx = int(i[N.SHARD_IT]), int(i[N.SHARD_ELL]), int(i[N.SHARD_MAX_ITERS])
        rr_new = float(red[0])
        beta = rr_new / float(state[N.SHARD_RR])
        rel = rr_new ** 0.5 / float(state[N.SHARD_NORM_B])
        cont = rel > float(state[N.SHARD_TOL]) and it < mx
        if k:
            mu = _chol_solve(chol, red[1:1 + k])
            p[:rows] = beta * p[:rows] + r[:rows] - w[:rows] @ mu
        else:
            p[:rows] = r[:rows] + beta * p[:rows]
        if cont and it < ell:
            log.p[it, :rows] = p[:rows]
            if k:
                log.mu[it, :k] = mu
        hist[it] = rel
        if it - 1 < ell:
            log.beta[it - 1] = beta
        state[N.SHARD_RR], state[N.SHARD_BETA], state[N.SHARD_REL] = rr_new, beta, rel
        i[N.SHARD_DONE] = 0 if cont else 1


# ---- symmetric sharded products (dcg_shard_rbf_sym_partial / dcg_shard_epilogue)
# The tile-share partition restated from csrc/symgemv.cuh (sym_cost4,
# sym_tile_begin): same integer arithmetic, so the CPU ranks cover exactly the
# tiles the CUDA ranks would.
TB = 64


def _side(n):
    return (n + TB - 1) // TB


def _row_base(i):
    return i * (i + 1) // 2


def _tile_row(t):
    i = int(((8 * t + 1) ** 0.5 - 1) * 0.5)
    while _row_base(i + 1) <= t:
        i += 1
    while _row_base(i) > t:
        i -= 1
    return i


def _cost4(t, n):
    nt = _side(n)
    last = _row_base(nt - 1) if n % TB else _row_base(nt)
    return 4 * t + max(t - last, 0) + 4 * _tile_row(t)


def tile_begin(n, parts, b):
    nt = _side(n)
    ntt = nt * (nt + 1) // 2
    if b <= 0:
        return 0
    if b >= parts:
        return ntt
    goal = (b * _cost4(ntt, n) + parts - 1) // parts
    lo, hi = 0, ntt
    while lo < hi:
        mid = (lo + hi) // 2
        if _cost4(mid, n) >= goal:
            hi = mid
        else:
            lo = mid + 1
    return lo


class CpuSymOperator:
    """A dense symmetric K standing in for the matrix-free operator's values:
    this rank's slab rows for the epilogue, its tile share for the product."""

    symmetric = True

    def __init__(self, kfull, row0, rows, rank, world, s=None, shift=0.0):
        self.kfull, self.n = kfull, int(kfull.shape[0])
        self.row0, self.rows, self.rank, self.world = int(row0), int(rows), int(rank), int(world)
        self.s, self.shift = s, float(shift)

    def scaled(self, s, shift):
        return CpuSymOperator(self.kfull, self.row0, self.rows, self.rank, self.world, s, shift)


def _sym_partial(self, op, vfull, t, state=None):
    if self._done(state):
        return
    n = op.n
    v = vfull[:n]
    sv = op.s * v if op.s is not None else v
    t[:n] = 0.0
    t_lo, t_hi = tile_begin(n, op.world, op.rank), tile_begin(n, op.world, op.rank + 1)
    for tid in range(t_lo, t_hi):
        i = _tile_row(tid)
        j = tid - _row_base(i)
        ri, rj = slice(i * TB, min(n, i * TB + TB)), slice(j * TB, min(n, j * TB + TB))
        blk = op.kfull[ri, rj]
        t[ri] += blk @ sv[rj]
        if j < i:
            t[rj] += blk.t() @ sv[ri]


def _epilogue(self, mode, op, vfull, b, t, out, part, state=None):
    if self._done(state):
        return
    r0, rows = op.row0, op.rows
    tr = t[r0:r0 + rows]
    if op.s is not None:
        tr = op.s[r0:r0 + rows] * tr
    ax = op.shift * vfull[r0:r0 + rows] + tr
    if mode == 0:
        out[:rows] = ax
        part[0] = torch.dot(vfull[r0:r0 + rows], ax)
    else:
        out[:rows] = b[:rows] - ax


CpuShardBackend.sym_partial = _sym_partial
CpuShardBackend.epilogue = _epilogue


class CpuTileShareOperator:
    """A dense symmetric K standing in for a stored tile share: this rank's
    slab rows (row0, rows) and share (rank, world) of the packed tiles; the
    solve runs on replicated vectors (sharded.sharded_solve's share path)."""

    def __init__(self, kfull, row0, rows, rank, world, s=None, shift=0.0):
        self.kfull, self.n = kfull, int(kfull.shape[0])
        self.row0, self.rows, self.rank, self.world = int(row0), int(rows), int(rank), int(world)
        self.share = (rank, world)
        self.s, self.shift = s, float(shift)

    def scaled(self, s, shift):
        return CpuTileShareOperator(self.kfull, self.row0, self.rows, self.rank, self.world, s, shift)


def _tiles_partial(self, op, vfull, t, state=None):
    _sym_partial(self, op, vfull, t, state)


def _epilogue_any(self, mode, op, vfull, b, t, out, part, state=None):
    if getattr(op, "share", None) is None:
        return _epilogue(self, mode, op, vfull, b, t, out, part, state)
    if self._done(state):
        return
    n = op.n
    tr = t[:n] if op.s is None else op.s[:n] * t[:n]
    ax = op.shift * vfull[:n] + tr
    if mode == 0:
        out[:n] = ax
        part[0] = torch.dot(vfull[:n], ax)
    else:
        out[:n] = b[:n] - ax


CpuShardBackend.tiles_partial = _tiles_partial
CpuShardBackend.epilogue = _epilogue_any
