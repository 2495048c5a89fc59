"""CPU, world_size 2 over gloo: the host logic of the row-sharded solver
(paper_1706_00241_b200/sharded.py) - partition, padded all-gather, the
collective sequence, device-state polling, the true-residual path and the
Krylov-log layout - against the reference algorithm (oracle).

The per-rank arithmetic runs through tests/shard_cpu_backend.py, a CPU
restatement of csrc/shard.cu; the CUDA kernels themselves are covered by the
GPU tests (test_gpu_sharded.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import random_spd
from oracle import defcg_oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(seed, n, k, kappa):
    rng = np.random.default_rng(seed)
    a = random_spd(rng, n, kappa=kappa)
    b = rng.standard_normal(n)
    xprev = rng.standard_normal(n) * 0.1
    w = rng.standard_normal((n, k)) if k else np.zeros((n, 0))
    return a, b, xprev, w


def _worker(rank, world, port, cases, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from shard_cpu_backend import CpuShardBackend

        from paper_1706_00241_b200 import SolverConfig
        from paper_1706_00241_b200.sharded import ShardBasis, ShardedOperator, TorchComm, row_range, sharded_solve

        comm, be = TorchComm(), CpuShardBackend()
        results = []
        for (seed, n, k, kappa, tol, ell, every, max_iters, zero_b) in cases:
            a, b, xprev, w = _case(seed, n, k, kappa)
            if zero_b:
                b = np.zeros(n)
            r0, rows = row_range(n, world, rank)
            t = lambda v: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
            op = ShardedOperator(t(a[r0:r0 + rows]), n, n, r0, rows)
            basis = None
            if k:
                aw = a @ w
                g = w.T @ aw
                basis = ShardBasis(t(w), t(aw), t(np.linalg.cholesky(0.5 * (g + g.T))))
            cfg = SolverConfig(tol=tol, ell=ell, recompute_residual_every=every, max_iters=max_iters)
            x, rep, log = sharded_solve(op, t(b[r0:r0 + rows]), t(xprev[r0:r0 + rows]), basis, cfg, comm, be, poll=3)
            parts = [torch.zeros(-(-n // world), dtype=torch.float64) for _ in range(world)]
            pad = torch.zeros(-(-n // world), dtype=torch.float64)
            pad[:rows] = x
            dist.all_gather(parts, pad)
            xfull = torch.cat(parts)[:n].numpy()
            # Krylov log on this rank's rows: r_j - r_{j+1} = alpha_j (A p_j)_rows
            m = log.m
            logok = True
            for j in range(min(m, 3)):
                pj = torch.zeros(-(-n // world) * world, dtype=torch.float64)
                comm.allgather(log.p[j, :rows], pj)
                apj = a[r0:r0 + rows] @ pj[:n].numpy()
                lhs = (log.r[j, :rows] - log.r[j + 1, :rows]).numpy()
                logok &= bool(np.allclose(lhs, float(log.alpha[j]) * apj, rtol=1e-8, atol=1e-10))
            results.append((xfull, rep.iterations, rep.residual_history, m, logok))
        if rank == 0:
            out.put(results)
    finally:
        dist.destroy_process_group()


CASES = [
    # seed, n, k, kappa, tol, ell, recompute_every, max_iters, zero_b
    # (kappa / tol keep every solve below n iterations, where CG counts are
    # not rounding-driven, so +-1 is the bar)
    (1, 91, 0, 1e2, 1e-9, 8, 0, None, False),      # CG, odd n (ragged last slab)
    (2, 96, 4, 1e2, 1e-9, 8, 5, None, False),      # def-CG with the true-residual path
    (3, 80, 3, 30.0, 1e-9, 20, 50, None, False),
    (4, 40, 2, 1e3, 1e-12, 4, 0, 7, False),        # max_iters stop
    (5, 33, 2, 1e2, 1e-10, 4, 0, None, True),      # zero right-hand side
]


def test_sharded_solver_world2_matches_reference():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, CASES, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for case, (x, its, hist, m, logok) in zip(CASES, results):
        seed, n, k, kappa, tol, ell, every, max_iters, zero_b = case
        a, b, xprev, w = _case(seed, n, k, kappa)
        if zero_b:
            b = np.zeros(n)
        cfg = O.Cfg(tol=tol, ell=ell, recompute_residual_every=every, max_iters=max_iters)
        if k:
            xr, rep, _ = O.deflated_cg_solve(a, b, xprev, O.refresh_basis(a, w, be="numpy"), cfg, be="numpy")
        else:
            xr, rep, _ = O.cg_solve(a, b, xprev, cfg, be="numpy")
        assert abs(its - rep.iterations) <= 1, (case, its, rep.iterations)
        if zero_b:
            assert its == 0 and hist == [0.0] and np.all(x == 0.0)
            continue
        assert np.linalg.norm(x - xr) <= 1e-7 * max(np.linalg.norm(xr), 1e-300), case
        assert abs(hist[0] - rep.residual_history[0]) <= 1e-12 * max(1.0, rep.residual_history[0])
        assert m == min(its, ell)
        assert logok, case
        if max_iters is not None:
            assert its == max_iters


def _sym_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from shard_cpu_backend import CpuShardBackend, CpuSymOperator

        from paper_1706_00241_b200 import SolverConfig
        from paper_1706_00241_b200.sharded import TorchComm, row_range, sharded_solve

        comm, be = TorchComm(), CpuShardBackend()
        results = []
        for seed, n in ((7, 150), (8, 200)):
            a, b, xprev, _ = _case(seed, n, 0, 50.0)
            t = lambda v: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
            r0, rows = row_range(n, world, rank)
            op = CpuSymOperator(t(a), r0, rows, rank, world)
            x, rep, _ = sharded_solve(op, t(b[r0:r0 + rows]), t(xprev[r0:r0 + rows]), None,
                                      SolverConfig(tol=1e-10, ell=6, recompute_residual_every=9), comm, be, poll=2)
            parts = [torch.zeros(-(-n // world), dtype=torch.float64) for _ in range(world)]
            pad = torch.zeros(-(-n // world), dtype=torch.float64)
            pad[:rows] = x
            dist.all_gather(parts, pad)
            results.append((torch.cat(parts)[:n].numpy(), rep.iterations))
        if rank == 0:
            out.put(results)
    finally:
        dist.destroy_process_group()


def test_symmetric_sharded_products_world2():
    """The symmetric sharded product path (each rank a share of the
    lower-triangle tiles, an all-reduce of K (s (.) p), the slab epilogue)
    through sharded_solve over gloo, world 2, against the reference CG; the
    true-residual path uses the same product."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sym_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (seed, n), (x, its) in zip(((7, 150), (8, 200)), results):
        a, b, xprev, _ = _case(seed, n, 0, 50.0)
        xr, rep, _ = O.cg_solve(a, b, xprev, O.Cfg(tol=1e-10, ell=6, recompute_residual_every=9), be="numpy")
        assert abs(its - rep.iterations) <= 1, (n, its, rep.iterations)
        assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)


def test_tile_share_partition_matches_device_rule():
    """The CPU restatement of the tile-share partition covers every tile once."""
    from shard_cpu_backend import _side, tile_begin

    for n in (1, 63, 64, 150, 1000, 5000):
        ntt = _side(n) * (_side(n) + 1) // 2
        for world in (1, 2, 3, 8):
            cuts = [tile_begin(n, world, b) for b in range(world + 1)]
            assert cuts[0] == 0 and cuts[-1] == ntt
            assert all(c0 <= c1 for c0, c1 in zip(cuts, cuts[1:]))


def test_row_partition_covers_rows():
    from paper_1706_00241_b200.sharded import row_block, row_range

    for n in (1, 7, 64, 65, 1000):
        for world in (1, 2, 3, 8):
            spans = [row_range(n, world, r) for r in range(world)]
            assert sum(rows for _, rows in spans) == n
            mb = row_block(n, world)
            for r, (r0, rows) in enumerate(spans):
                assert rows <= mb and (rows == 0 or r0 == r * mb)


def _share_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from shard_cpu_backend import CpuShardBackend, CpuTileShareOperator

        from paper_1706_00241_b200 import SolverConfig
        from paper_1706_00241_b200.sharded import ShardBasis, TorchComm, row_range, sharded_solve

        comm, be = TorchComm(), CpuShardBackend()
        results = []
        for seed, n, k in ((11, 150, 0), (12, 200, 4), (13, 131, 3)):
            a, b, xprev, w = _case(seed, n, k, 50.0)
            t = lambda v: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
            r0, rows = row_range(n, world, rank)
            op = CpuTileShareOperator(t(a), r0, rows, rank, world)
            basis = None
            if k:
                aw = a @ w
                g = w.T @ aw
                basis = ShardBasis(t(w), t(aw), t(np.linalg.cholesky(0.5 * (g + g.T))))
            x, rep, log = sharded_solve(op, t(b[r0:r0 + rows]), t(xprev[r0:r0 + rows]), basis,
                                        SolverConfig(tol=1e-10, ell=6, recompute_residual_every=9), comm, be, poll=2)
            assert log.replicated and log.r.shape[1] == n   # the log holds all rows on every rank
            parts = [torch.zeros(-(-n // world), dtype=torch.float64) for _ in range(world)]
            pad = torch.zeros(-(-n // world), dtype=torch.float64)
            pad[:rows] = x
            dist.all_gather(parts, pad)
            results.append((torch.cat(parts)[:n].numpy(), rep.iterations))
        if rank == 0:
            out.put(results)
    finally:
        dist.destroy_process_group()


def test_tile_share_solver_world2():
    """The stored tile-share path (each rank its share of the lower-triangle
    tiles, replicated vectors, one all-reduce of K (s (.) p) per product;
    everything else redundant on every rank) through sharded_solve over gloo,
    world 2, CG and def-CG with the true-residual path, against the reference."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_share_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (seed, n, k), (x, its) in zip(((11, 150, 0), (12, 200, 4), (13, 131, 3)), results):
        a, b, xprev, w = _case(seed, n, k, 50.0)
        cfg = O.Cfg(tol=1e-10, ell=6, recompute_residual_every=9)
        if k:
            basis = O.refresh_basis(a, w)
            xr, rep, _ = O.deflated_cg_solve(a, b, xprev, basis, cfg, be="numpy")
        else:
            xr, rep, _ = O.cg_solve(a, b, xprev, cfg, be="numpy")
        assert abs(its - rep.iterations) <= 1, (n, k, its, rep.iterations)
        assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)
