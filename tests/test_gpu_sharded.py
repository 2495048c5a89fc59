"""GPU: the row-sharded def-CG kernels (csrc/shard.cu, include/defcg_b200.h L5)
through the sharded driver (paper_1706_00241_b200/sharded.py).

* world = 1: same answers as the single-GPU persistent solver;
* two ranks in one process: each rank is a thread with its own library
  context, the collectives are host-ordered copies on the one stream (the
  kernels never wait on each other), checked against the reference (oracle);
* a recycled sequence (refresh -> solve -> extraction on gathered data)
  against the single-GPU solve_next."""

import threading

import numpy as np
import pytest
import torch

from conftest import random_spd
from oracle import defcg_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1706_00241_b200 as P

    return P


class ThreadComm:
    """In-process collectives for `world` rank threads sharing one device."""

    def __init__(self, shared, rank, world):
        self.shared, self.rank, self.world = shared, rank, world

    def _barrier(self):
        self.shared["barrier"].wait()

    def allgather(self, local, full):
        mb = full.shape[0] // self.world
        self.shared.setdefault("slots", {})
        self._barrier()
        self.shared["slots"][self.rank] = local.clone()
        self._barrier()
        for r in range(self.world):
            src = self.shared["slots"][r]
            full[r * mb: r * mb + src.shape[0]].copy_(src)
        self._barrier()

    def allreduce(self, buf):
        self.shared.setdefault("red", {})
        self._barrier()
        self.shared["red"][self.rank] = buf.clone()
        self._barrier()
        acc = self.shared["red"][0].clone()
        for r in range(1, self.world):
            acc += self.shared["red"][r]
        buf.copy_(acc)
        self._barrier()
        return buf


def run_ranks(world, fn):
    shared = {"barrier": threading.Barrier(world)}
    out, errs = [None] * world, []

    def body(rank):
        try:
            out[rank] = fn(rank, ThreadComm(shared, rank, world))
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errs.append(e)
            shared["barrier"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


def slab_op(a, world, rank, P):
    from paper_1706_00241_b200 import _device as D
    from paper_1706_00241_b200.sharded import ShardedOperator, row_range

    n = a.shape[0]
    r0, rows = row_range(n, world, rank)
    ld = D.padded_ld(n)
    slab = torch.zeros(max(rows, 1), ld, dtype=torch.float64, device="cuda")
    slab[:rows, :n] = torch.from_numpy(a[r0:r0 + rows])
    return ShardedOperator(slab, n, ld, r0, rows)


def dev(v):
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).cuda()


@pytest.mark.parametrize("k,every", [(0, 0), (5, 0), (5, 7)])
def test_world1_matches_single_gpu_solver(P, rng, k, every):
    from paper_1706_00241_b200.sharded import SelfComm, ShardBasis, sharded_solve

    n = 300
    a = random_spd(rng, n, kappa=100.0)   # converges well below n iterations
    b = rng.standard_normal(n)
    xprev = 0.1 * rng.standard_normal(n)
    cfg = P.SolverConfig(tol=1e-10, ell=10, recompute_residual_every=every)
    basis = P.refresh_basis(a, rng.standard_normal((n, k))) if k else None
    if k:
        x_ref, rep_ref, _ = P.deflated_cg_solve(a, b, xprev, basis, cfg)
        sb = ShardBasis(basis.w_dev, basis.aw_dev, basis.chol_dev)
    else:
        x_ref, rep_ref, _ = P.cg_solve(a, b, xprev, cfg)
        sb = None
    x, rep, log = sharded_solve(slab_op(a, 1, 0, P), dev(b), dev(xprev), sb, cfg, SelfComm())
    assert abs(rep.iterations - rep_ref.iterations) <= 1
    xs = x.cpu().numpy()
    assert np.linalg.norm(xs - x_ref) <= 1e-8 * np.linalg.norm(x_ref)
    assert log.m == min(rep.iterations, 10)
    assert abs(rep.residual_history[0] - rep_ref.residual_history[0]) <= 1e-12 * rep_ref.residual_history[0]


@pytest.mark.parametrize("k,every,n", [(0, 0, 300), (5, 0, 300), (5, 7, 300), (32, 0, 2500)])
def test_tile_share_fused_step_is_bitwise_the_three_launch_path(P, rng, monkeypatch, k, every, n):
    """dcg_shard_step (epilogue + update + direction in one cooperative
    launch) against the three separate launches: same partitions and
    summation orders, so x, the residual history and the Krylov log agree bit
    for bit (also across a true-residual refresh, which takes the separate
    launches in both runs)."""
    from paper_1706_00241_b200.sharded import SelfComm, ShardBasis, sharded_solve

    a = random_spd(rng, n, kappa=100.0)
    b = rng.standard_normal(n)
    xprev = 0.1 * rng.standard_normal(n)
    cfg = P.SolverConfig(tol=1e-10, ell=10, recompute_residual_every=every)
    sb = None
    if k:
        basis = P.refresh_basis(a, rng.standard_normal((n, k)))
        sb = ShardBasis(basis.w_dev, basis.aw_dev, basis.chol_dev)
    op = share_op(a, 1, 0, P)
    out = []
    for fused in (True, False):
        if fused:
            monkeypatch.delenv("DCG_SHARD_NO_FUSED_STEP", raising=False)
        else:
            monkeypatch.setenv("DCG_SHARD_NO_FUSED_STEP", "1")
        x, rep, log = sharded_solve(op, dev(b), dev(xprev), sb, cfg, SelfComm())
        m = log.m
        out.append((x.cpu().numpy(), np.array(rep.residual_history), log.p[:m].cpu().numpy(), log.r[:m + 1].cpu().numpy(),
                    log.alpha[:m].cpu().numpy(), log.beta[:m].cpu().numpy(),
                    log.mu[:m].cpu().numpy() if k else np.zeros(0)))
    assert len(out[0][1]) == len(out[1][1]) and len(out[0][1]) > 5
    for u, v in zip(out[0], out[1]):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("world,k,every", [(2, 0, 0), (2, 4, 0), (3, 4, 6)])
def test_virtual_ranks_match_reference(P, rng, world, k, every):
    from paper_1706_00241_b200.sharded import DeviceShardBackend, ShardBasis, sharded_solve

    n = 257
    a = random_spd(rng, n, kappa=100.0)
    b = rng.standard_normal(n)
    xprev = 0.1 * rng.standard_normal(n)
    w = rng.standard_normal((n, k))
    cfg = P.SolverConfig(tol=1e-10, ell=8, recompute_residual_every=every)
    ocfg = O.Cfg(tol=1e-10, ell=8, recompute_residual_every=every)
    if k:
        ob = O.refresh_basis(a, w, be="numpy")
        x_ref, rep_ref, _ = O.deflated_cg_solve(a, b, xprev, ob, ocfg, be="numpy")
        aw = a @ w
        g = w.T @ aw
        sb = ShardBasis(dev(w), dev(aw), dev(np.linalg.cholesky(0.5 * (g + g.T))))
    else:
        x_ref, rep_ref, _ = O.cg_solve(a, b, xprev, ocfg, be="numpy")
        sb = None

    def rank_fn(rank, comm):
        op = slab_op(a, world, rank, P)
        r0, rows = op.row0, op.rows
        x, rep, _ = sharded_solve(op, dev(b[r0:r0 + rows]), dev(xprev[r0:r0 + rows]), sb, cfg, comm,
                                  DeviceShardBackend(slot=2 + rank), poll=3)
        torch.cuda.synchronize()
        return r0, x.cpu().numpy(), rep

    outs = run_ranks(world, rank_fn)
    x = np.zeros(n)
    for r0, xl, _ in outs:
        x[r0:r0 + xl.shape[0]] = xl
    reps = [o[2] for o in outs]
    assert all(r.iterations == reps[0].iterations for r in reps)          # ranks agree
    assert all(r.residual_history == reps[0].residual_history for r in reps)
    assert abs(reps[0].iterations - rep_ref.iterations) <= 1
    assert np.linalg.norm(x - x_ref) <= 1e-8 * np.linalg.norm(x_ref)


def test_sharded_sequence_matches_single_gpu(P, rng):
    """solve_next over a drifting sequence A_i = A + i * 0.05 I: same
    iteration counts (+-1) as the single-GPU sequence, solutions 1e-8."""
    from paper_1706_00241_b200.sharded import SelfComm, ShardSequenceState, sharded_solve_next

    n = 400
    a0 = random_spd(rng, n, kappa=30.0)   # ~50-iteration solves: counts not rounding-driven
    bs = [rng.standard_normal(n) for _ in range(4)]
    cfg = P.SolverConfig(tol=1e-9, ell=12)
    st = P.SequenceState(k=6, cfg=cfg, selection="largest")
    sst = ShardSequenceState(k=6, cfg=cfg, selection="largest")
    for i, b in enumerate(bs):
        a = a0 + 0.05 * i * np.eye(n)
        x_ref, st = P.solve_next(st, a, b)
        x, sst = sharded_solve_next(sst, slab_op(a, 1, 0, P), dev(b), SelfComm())
        assert abs(sst.history[-1].iterations - st.history[-1].iterations) <= 1, (i, sst.history[-1].iterations,
                                                                                    st.history[-1].iterations)
        assert np.linalg.norm(x.cpu().numpy() - x_ref) <= 1e-8 * np.linalg.norm(x_ref)


def test_sharded_sequence_keeps_the_basis_on_the_device(P, rng, monkeypatch):
    """The sharded sequence hands W_next / AW_next from the extraction to the
    next refresh as device tensors: the RitzExtraction's numpy properties (a
    device -> host copy each; 2 x 12.8 MB per step at config 3) must not be
    touched on that path."""
    from paper_1706_00241_b200 import recycle as R
    from paper_1706_00241_b200.sharded import SelfComm, ShardSequenceState, sharded_solve_next

    def boom(self):
        raise AssertionError("host copy of the next basis on the sharded path")

    for name in ("w_next", "aw_next", "z", "u", "theta"):
        monkeypatch.setattr(R.RitzExtraction, name, property(boom))
    n = 300
    a0 = random_spd(rng, n, kappa=30.0)
    cfg = P.SolverConfig(tol=1e-9, ell=10)
    sst = ShardSequenceState(k=5, cfg=cfg, selection="largest")
    for i in range(3):
        a = a0 + 0.05 * i * np.eye(n)
        _, sst = sharded_solve_next(sst, slab_op(a, 1, 0, P), dev(rng.standard_normal(n)), SelfComm())
    assert sst.basis is not None and sst.basis.k == 5 and sst.basis.w.is_cuda


def test_sharded_laplace_newton_world1_matches_gpc(P):
    """The sharded GPC Newton driver at world = 1 against laplace_newton on
    the config-1 inputs: iteration counts +-1 per step, psi within 1e-8."""
    from paper_1706_00241_b200.sharded import SelfComm, sharded_laplace_newton

    x, y = O.gpc_inputs(2000, 5, 0)
    cfg = P.SolverConfig(tol=1e-8, ell=12)
    gram = P.rbf_kernel(x, P.KernelParams(1.0, 1.5))
    _, recs = P.laplace_newton(gram, y, "defcg", cfg, newton_tol=-np.inf, max_newton=6, k=8, selection="largest")
    srecs = sharded_laplace_newton(x, y, P.KernelParams(1.0, 1.5), cfg, newton_tol=-np.inf, max_newton=6, k=8,
                                   selection="largest", comm=SelfComm())
    assert len(srecs) == len(recs)
    for a, b in zip(srecs, recs):
        assert abs(a.solver_iterations - b.solver_iterations) <= 1, ([r.solver_iterations for r in srecs],
                                                                     [r.solver_iterations for r in recs])
        assert abs(a.psi - b.psi) <= 1e-8 * abs(b.psi)
    assert np.linalg.norm(srecs[-1].f - recs[-1].f) <= 1e-6 * np.linalg.norm(recs[-1].f)


def test_matrix_free_slab_products_match_stored(P, rng):
    """Config-5 building block: the matrix-free slab operator (row-owned
    tensor-pipe kernel) against the stored slab's products, single vector
    (the sharded solve's apply) and multi-vector (its refresh), on row slabs
    that are not 64-aligned."""
    from paper_1706_00241_b200.sharded import row_range, sharded_rbf_kernel

    n, dim = 900, 9
    x = torch.from_numpy(rng.standard_normal((n, dim))).cuda()
    params = P.KernelParams(1.2, 1.7)
    s = torch.from_numpy(rng.uniform(0.2, 0.6, n)).cuda()
    v = torch.from_numpy(rng.standard_normal(n)).cuda()
    w = torch.from_numpy(rng.standard_normal((n, 11))).cuda()

    class C:
        def __init__(self, rank, world):
            self.rank, self.world = rank, world

    for world in (1, 3):
        for rank in range(world):
            st = sharded_rbf_kernel(x, params, comm=C(rank, world)).scaled(s, 1.0)
            mf = sharded_rbf_kernel(x, params, comm=C(rank, world), matrix_free=True).scaled(s, 1.0)
            r0, rows = row_range(n, world, rank)
            for a in (st, mf):
                assert (a.row0, a.rows) == (r0, rows)
            outs = []
            for a in (st, mf):
                y = torch.empty(rows, dtype=torch.float64, device="cuda")
                yb = torch.empty(rows, 11, dtype=torch.float64, device="cuda")
                c = a.c_struct()
                import ctypes

                P._native.check(P._native.lib().dcg_op_apply(P._device.ctx(), P._device.stream(), ctypes.byref(c),
                                                             v.data_ptr(), y.data_ptr()))
                P._native.check(P._native.lib().dcg_op_apply_block(P._device.ctx(), P._device.stream(),
                                                                   ctypes.byref(c), w.data_ptr(), 11, yb.data_ptr()))
                outs.append((y, yb))
            for ref, got in zip(outs[0], outs[1]):
                err = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
                assert err <= 1e-13, (world, rank, err)


def test_sharded_laplace_newton_matrix_free(P):
    """The sharded Newton driver on the matrix-free slab (config 5's path) at
    world = 1 against laplace_newton on the stored Gram: iteration counts +-1,
    psi within 1e-8."""
    from paper_1706_00241_b200.sharded import SelfComm, sharded_laplace_newton

    x, y = O.gpc_inputs(1500, 6, 0)
    cfg = P.SolverConfig(tol=1e-8, ell=12)
    gram = P.rbf_kernel(x, P.KernelParams(1.0, 1.5))
    _, recs = P.laplace_newton(gram, y, "defcg", cfg, newton_tol=-np.inf, max_newton=4, k=8, selection="largest")
    srecs = sharded_laplace_newton(x, y, P.KernelParams(1.0, 1.5), cfg, newton_tol=-np.inf, max_newton=4, k=8,
                                   selection="largest", comm=SelfComm(), matrix_free=True)
    for a, b in zip(srecs, recs):
        assert abs(a.solver_iterations - b.solver_iterations) <= 1
        assert abs(a.psi - b.psi) <= 1e-8 * abs(b.psi)


@pytest.mark.parametrize("world,k", [(1, 0), (2, 0), (3, 5)])
def test_symmetric_matrix_free_virtual_ranks(P, rng, world, k):
    """Config 5's sharded product in the symmetric form: each rank evaluates
    its share of the lower-triangle tiles of the regenerated K and the ranks
    all-reduce K (s (.) p).  Against the single-GPU solve on the stored Gram
    of the same points: same iterations (+-1), solutions 1e-9."""
    from paper_1706_00241_b200.sharded import DeviceShardBackend, ShardBasis, sharded_rbf_kernel, sharded_solve

    n, dim = 700, 5
    x = rng.standard_normal((n, dim))
    params = P.KernelParams(1.0, 1.4)
    s = rng.uniform(0.2, 0.5, n)
    b = rng.standard_normal(n)
    xprev = 0.05 * rng.standard_normal(n)
    cfg = P.SolverConfig(tol=1e-10, ell=8)
    a_st = P.rbf_kernel(dev(x), params).scaled(dev(s), 1.0)
    if k:
        w = rng.standard_normal((n, k))
        basis = P.refresh_basis(a_st, w)
        x_ref, rep_ref, _ = P.deflated_cg_solve(a_st, b, xprev, basis, cfg)
        sb = ShardBasis(basis.w_dev, basis.aw_dev, basis.chol_dev.contiguous())
    else:
        x_ref, rep_ref, _ = P.cg_solve(a_st, b, xprev, cfg)
        sb = None

    def rank_fn(rank, comm):
        op = sharded_rbf_kernel(dev(x), params, comm=comm, matrix_free=True).scaled(dev(s), 1.0)
        assert op.symmetric
        r0, rows = op.row0, op.rows
        xl, rep, _ = sharded_solve(op, dev(b[r0:r0 + rows]), dev(xprev[r0:r0 + rows]), sb, cfg, comm,
                                   DeviceShardBackend(slot=2 + rank), poll=3)
        torch.cuda.synchronize()
        return r0, xl.cpu().numpy(), rep

    outs = run_ranks(world, rank_fn)
    xs = np.zeros(n)
    for r0, xl, _ in outs:
        xs[r0:r0 + xl.shape[0]] = xl
    reps = [o[2] for o in outs]
    assert all(r.iterations == reps[0].iterations for r in reps)
    assert abs(reps[0].iterations - rep_ref.iterations) <= 1, (reps[0].iterations, rep_ref.iterations)
    assert np.linalg.norm(xs - x_ref) <= 1e-9 * np.linalg.norm(x_ref)


# ---------------------------------------------------------------------------
# stored tile shares (replicated vectors, one all-reduce per product)
# ---------------------------------------------------------------------------


def share_op(a, world, rank, P):
    """The rank's row slab plus its share of the packed tiles of a dense matrix."""
    import ctypes

    from paper_1706_00241_b200 import _device as D
    from paper_1706_00241_b200 import _native as N
    from paper_1706_00241_b200.sharded import TileShare, tile_range

    op = slab_op(a, world, rank, P)
    n = a.shape[0]
    kfull, ld = D.to_dev_padded(np.ascontiguousarray(a))
    kp = D.empty(int(N.lib().dcg_packed_sym_doubles(n)))
    N.check(N.lib().dcg_pack_sym(D.ctx(), D.stream(), kfull.data_ptr(), ld, n, kp.data_ptr()))
    t_lo, t_hi = tile_range(n, world, rank)
    op.share = TileShare(kp[t_lo * 4096:t_hi * 4096].clone(), t_lo, t_hi, rank, world)
    del ctypes
    return op


@pytest.mark.parametrize("k,every", [(0, 0), (5, 0), (5, 7)])
def test_tile_share_world1_matches_single_gpu_solver(P, rng, k, every):
    from paper_1706_00241_b200.sharded import SelfComm, ShardBasis, sharded_solve

    n = 300
    a = random_spd(rng, n, kappa=100.0)
    b = rng.standard_normal(n)
    xprev = 0.1 * rng.standard_normal(n)
    cfg = P.SolverConfig(tol=1e-10, ell=10, recompute_residual_every=every)
    basis = P.refresh_basis(a, rng.standard_normal((n, k))) if k else None
    if k:
        x_ref, rep_ref, _ = P.deflated_cg_solve(a, b, xprev, basis, cfg)
        sb = ShardBasis(basis.w_dev, basis.aw_dev, basis.chol_dev)
    else:
        x_ref, rep_ref, _ = P.cg_solve(a, b, xprev, cfg)
        sb = None
    x, rep, log = sharded_solve(share_op(a, 1, 0, P), dev(b), dev(xprev), sb, cfg, SelfComm())
    assert log.replicated
    assert abs(rep.iterations - rep_ref.iterations) <= 1
    assert np.linalg.norm(x.cpu().numpy() - x_ref) <= 1e-8 * np.linalg.norm(x_ref)


@pytest.mark.parametrize("world,k,every", [(2, 0, 0), (2, 4, 0), (3, 4, 6)])
def test_tile_share_virtual_ranks_match_reference(P, rng, world, k, every):
    from paper_1706_00241_b200.sharded import DeviceShardBackend, ShardBasis, sharded_solve

    n = 1000   # 16 tile rows: several ranks' shares cut tile rows mid-way
    a = O.rbf_kernel(rng.standard_normal((n, 4)), 1.0, 0.9) + 0.5 * np.eye(n)
    b = rng.standard_normal(n)
    xprev = 0.1 * rng.standard_normal(n)
    w = rng.standard_normal((n, k))
    cfg = P.SolverConfig(tol=1e-10, ell=8, recompute_residual_every=every)
    ocfg = O.Cfg(tol=1e-10, ell=8, recompute_residual_every=every)
    if k:
        ob = O.refresh_basis(a, w, be="numpy")
        x_ref, rep_ref, _ = O.deflated_cg_solve(a, b, xprev, ob, ocfg, be="numpy")
        aw = a @ w
        g = w.T @ aw
        sb = ShardBasis(dev(w), dev(aw), dev(np.linalg.cholesky(0.5 * (g + g.T))))
    else:
        x_ref, rep_ref, _ = O.cg_solve(a, b, xprev, ocfg, be="numpy")
        sb = None

    def rank_fn(rank, comm):
        op = share_op(a, world, rank, P)
        r0, rows = op.row0, op.rows
        x, rep, _ = sharded_solve(op, dev(b[r0:r0 + rows]), dev(xprev[r0:r0 + rows]), sb, cfg, comm,
                                  DeviceShardBackend(slot=2 + rank), poll=3)
        torch.cuda.synchronize()
        return r0, x.cpu().numpy(), rep

    outs = run_ranks(world, rank_fn)
    x = np.zeros(n)
    for r0, xl, _ in outs:
        x[r0:r0 + xl.shape[0]] = xl
    reps = [o[2] for o in outs]
    assert all(r.iterations == reps[0].iterations for r in reps)
    assert all(r.residual_history == reps[0].residual_history for r in reps)
    assert abs(reps[0].iterations - rep_ref.iterations) <= 1
    assert np.linalg.norm(x - x_ref) <= 1e-8 * np.linalg.norm(x_ref)


@pytest.mark.parametrize("n,world", [(1000, 3), (777, 2)])
def test_packed_share_built_from_points_is_the_gram(P, rng, n, world):
    """dcg_k_rbf_gram_packed (a rank's tiles straight from X) is bitwise the
    packed copy of the stored Gram."""
    from paper_1706_00241_b200.sharded import sharded_rbf_kernel, tile_range

    x = rng.standard_normal((n, 6))
    params = P.KernelParams(1.3, 1.1)
    from paper_1706_00241_b200 import _device as D
    from paper_1706_00241_b200 import _native as N

    gram = P.rbf_kernel(dev(x), params)
    full = D.empty(int(N.lib().dcg_packed_sym_doubles(n)))   # pack_sym of the row-major Gram
    N.check(N.lib().dcg_pack_sym(D.ctx(), D.stream(), gram.kbuf.data_ptr(), gram.ldk, n, full.data_ptr()))

    class C:
        def __init__(self, rank, world):
            self.rank, self.world = rank, world

    for rank in range(world):
        op = sharded_rbf_kernel(dev(x), params, comm=C(rank, world))
        t_lo, t_hi = tile_range(n, world, rank)
        assert (op.share.t_lo, op.share.t_hi) == (t_lo, t_hi)
        assert torch.equal(op.share.kp, full[t_lo * 4096:t_hi * 4096])


def test_tile_share_laplace_newton_config3_recipe_virtual_ranks(P):
    """Config 3's recipe (d = 8, lengthscale 2, k = 32, ell_log = 36) at
    n = 3000 on two virtual ranks with tile shares: the sharded Newton driver
    against the reference (oracle), iterations +-1, psi 1e-8."""
    from paper_1706_00241_b200.sharded import DeviceShardBackend, sharded_laplace_newton

    n = 3000
    x, y = O.gpc_inputs(n, 8, 0)
    cfg = P.SolverConfig(tol=1e-8, ell=36)
    kmat = O.rbf_kernel(x, 1.0, 2.0)
    _, _, ref = O.laplace_newton(kmat, y, "defcg", O.Cfg(tol=1e-8, ell=36), newton_tol=-np.inf, max_newton=3, k=32,
                                 selection="largest", be="numpy")

    def rank_fn(rank, comm):
        recs = sharded_laplace_newton(x, y, P.KernelParams(1.0, 2.0), cfg, newton_tol=-np.inf, max_newton=3, k=32,
                                      selection="largest", comm=comm, backend=DeviceShardBackend(slot=2 + rank))
        torch.cuda.synchronize()
        return recs

    outs = run_ranks(2, rank_fn)
    for recs in outs:
        assert [r.solver_iterations for r in recs] == [r.solver_iterations for r in outs[0]]
        for a, b in zip(recs, ref):
            assert abs(a.solver_iterations - b.solver_iterations) <= 1, ([r.solver_iterations for r in recs],
                                                                         [r.solver_iterations for r in ref])
            assert abs(a.psi - b.psi) <= 1e-8 * abs(b.psi)
