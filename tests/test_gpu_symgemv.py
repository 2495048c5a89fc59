"""GPU: the lower-triangle ("sym") product strategy against the full-row
strategy and an fp64 host product, over sizes that exercise partial edge
tiles, tiny systems (more CTAs than tiles) and the persistent solve kernel."""

import numpy as np
import pytest

from conftest import random_spd
from oracle import defcg_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1706_00241_b200 as P

    return P


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 130, 257, 1000, 2049, 5000])
def test_sym_matvec_matches_rows_and_host(P, n):
    rng = np.random.default_rng(n)
    a = random_spd(rng, n, 1e3) if n <= 1000 else O.rbf_kernel(rng.standard_normal((n, 4)), 1.0, 1.3)
    op = P.DenseOperator.from_matrix(a)
    assert op.strategy == "auto"
    op = op.with_strategy("sym")
    ak = np.asarray(op.kernel_view())     # exactly symmetric device copy
    assert np.array_equal(ak, ak.T)
    x = rng.standard_normal(n)
    s = rng.uniform(0.2, 0.6, n)
    for shift, sv in ((0.0, None), (1.0, s)):
        A = op.scaled(sv, shift)
        y_sym = A @ x
        y_rows = A.with_strategy("rows") @ x
        ref = (ak * np.outer(s, s) + np.eye(n)) @ x if sv is not None else ak @ x
        scale = (np.abs(ak) @ np.abs(x)) + 1.0
        assert np.all(np.abs(y_sym - ref) <= 64 * np.finfo(float).eps * scale)
        assert np.all(np.abs(y_sym - y_rows) <= 64 * np.finfo(float).eps * scale)
        assert np.array_equal(y_sym, A @ x)   # deterministic


@pytest.mark.parametrize("n,k", [(777, 0), (777, 12), (3000, 16)])
def test_sym_solve_matches_rows(P, n, k):
    rng = np.random.default_rng(7 + n + k)
    x = rng.standard_normal((n, 6))
    kmat = O.rbf_kernel(x, 1.0, 1.4)
    gram = P.DenseOperator.from_matrix(kmat).with_strategy("sym")
    s = rng.uniform(0.1, 0.5, n)
    A = gram.scaled(s, 1.0)
    b = rng.standard_normal(n)
    cfg = P.SolverConfig(tol=1e-10, ell=k + 4)
    if k:
        w = rng.standard_normal((n, k))
        bs = P.refresh_basis(A, w)
        br = P.refresh_basis(A.with_strategy("rows"), w)
        xs, rs, _ = P.deflated_cg_solve(A, b, np.zeros(n), bs, cfg)
        xr, rr, _ = P.deflated_cg_solve(A.with_strategy("rows"), b, np.zeros(n), br, cfg)
    else:
        xs, rs, _ = P.cg_solve(A, b, None, cfg)
        xr, rr, _ = P.cg_solve(A.with_strategy("rows"), b, None, cfg)
    assert abs(rs.iterations - rr.iterations) <= 1
    assert np.linalg.norm(xs - xr) / np.linalg.norm(xr) <= 1e-9
    dense = kmat * np.outer(s, s) + np.eye(n)
    assert np.linalg.norm(b - dense @ xs) / np.linalg.norm(b) <= 2e-10


@pytest.mark.parametrize("n", [1, 63, 64, 65, 257, 2049, 5000])
def test_packed_tiles_bitwise_rowmajor(P, n):
    """The packed tile copy (dcg_pack_sym, one bulk copy per tile) gives
    bitwise the products of the row-major lower-triangle tiles."""
    import torch

    rng = np.random.default_rng(100 + n)
    a = O.rbf_kernel(rng.standard_normal((n, 4)), 1.0, 1.3)
    op = P.DenseOperator.from_matrix(a).with_strategy("sym")
    rm = op.with_strategy("sym_rowmajor")
    assert P._native.lib().dcg_packed_sym_doubles(n) == ((n + 63) // 64) * ((n + 63) // 64 + 1) // 2 * 4096
    x = rng.standard_normal(n)
    s = rng.uniform(0.2, 0.6, n)
    for shift, sv in ((0.0, None), (1.0, s)):
        assert np.array_equal(op.scaled(sv, shift) @ x, rm.scaled(sv, shift) @ x)
    # the packed copy holds the swizzled lower triangle, zero beyond n
    buf = op._packed.buf.cpu().numpy().reshape(-1, 64, 64)
    nt = (n + 63) // 64
    t = nt * (nt + 1) // 2 - 1          # last (diagonal, edge) tile
    r = np.arange(64)[:, None]
    c = np.arange(64)[None, :]
    swz = r * 64 + 2 * ((c // 2) ^ ((r // 2) % 32)) + c % 2
    tile = buf[t].reshape(-1)[swz]
    kpad = np.zeros((nt * 64, nt * 64))
    kpad[:n, :n] = a
    assert np.array_equal(tile, kpad[(nt - 1) * 64:, (nt - 1) * 64:])
    del torch


@pytest.mark.parametrize("n,k,recompute", [(4500, 0, 0), (4500, 16, 0), (5000, 12, 7)])
def test_packed_solve_bitwise_rowmajor(P, n, k, recompute):
    """Persistent solve on the packed tiles (next pass's tiles issued before
    the grid barriers) against the row-major symmetric path: the same
    iterations and bitwise the same solution, with and without deflation and
    true-residual refreshes (extra products between iterations)."""
    rng = np.random.default_rng(11 + n + k)
    x = rng.standard_normal((n, 6))
    gram = P.DenseOperator.from_matrix(O.rbf_kernel(x, 1.0, 1.4)).with_strategy("sym")
    s = rng.uniform(0.1, 0.5, n)
    A = gram.scaled(s, 1.0)
    R = A.with_strategy("sym_rowmajor")
    b = rng.standard_normal(n)
    cfg = P.SolverConfig(tol=1e-10, ell=k + 4, recompute_residual_every=recompute)
    if k:
        w = rng.standard_normal((n, k))
        x0 = rng.standard_normal(n)
        basis = P.refresh_basis(A, w)   # one basis for both (its A W comes from the packed block product)
        xs, rs, _ = P.deflated_cg_solve(A, b, x0, basis, cfg)
        xr, rr, _ = P.deflated_cg_solve(R, b, x0, basis, cfg)
    else:
        xs, rs, _ = P.cg_solve(A, b, None, cfg)
        xr, rr, _ = P.cg_solve(R, b, None, cfg)
    assert rs.iterations == rr.iterations
    assert np.array_equal(xs, xr)
    assert np.array_equal(rs.residual_history, rr.residual_history)


@pytest.mark.parametrize("n,k", [(1, 1), (63, 3), (64, 16), (65, 7), (257, 16), (1000, 12), (2049, 16), (4500, 16),
                                 (3000, 24), (1000, 28), (4500, 32), (130, 33)])
def test_symmetric_block_product(P, n, k):
    """A W over the packed tiles (symblock.cu: each tile feeds K_IJ W_J and
    K_IJ' W_I on the FP64 tensor pipe; k <= 32, padded to 16 or 32 columns)
    against the row-major DMMA product and an fp64 host product; k = 24 and
    k = 33 take the row-major path."""
    rng = np.random.default_rng(300 + n + k)
    a = O.rbf_kernel(rng.standard_normal((n, 5)), 1.0, 1.2)
    op = P.DenseOperator.from_matrix(a).with_strategy("sym")
    w = rng.standard_normal((n, k))
    s = rng.uniform(0.2, 0.6, n)
    for shift, sv in ((0.0, None), (1.0, s)):
        A = op.scaled(sv, shift)
        y_sym = A @ w
        y_rows = A.with_strategy("rows") @ w
        ref = (a * np.outer(s, s) + np.eye(n)) @ w if sv is not None else a @ w
        scale = np.abs(a) @ np.abs(w) + 1.0
        assert np.all(np.abs(y_sym - ref) <= 64 * np.finfo(float).eps * scale)
        assert np.all(np.abs(y_sym - y_rows) <= 64 * np.finfo(float).eps * scale)
        assert np.array_equal(y_sym, A @ w)   # deterministic (units are drawn dynamically)


@pytest.mark.parametrize("n", [4096, 5000])
def test_rbf_kernel_packed_only(P, n):
    """rbf_kernel above SYM_MIN_N keeps only the packed tiles (built from X):
    they equal pack_sym of the row-major Gram, which is built only when asked
    for (here by .kbuf) and equals the direct builder; products, a solve and a
    k = 24 block product (which needs the rows) agree bitwise with an operator
    that has both copies."""
    import torch

    from paper_1706_00241_b200 import _device as D
    from paper_1706_00241_b200 import _native as N

    rng = np.random.default_rng(n)
    x = torch.from_numpy(rng.standard_normal((n, 6))).cuda()
    params = P.KernelParams(1.0, 1.3)
    g = P.rbf_kernel(x, params)
    assert g._packed.buf is not None and not g._rm.ready
    v = torch.from_numpy(rng.standard_normal(n)).cuda()
    s = torch.from_numpy(rng.uniform(0.2, 0.6, n)).cuda()
    A = g.scaled(s, 1.0)
    y_packed_only = A.matvec_dev(v).clone()
    w16 = torch.from_numpy(rng.standard_normal((n, 16))).cuda()
    yb16 = A.apply_block_dev(w16).clone()
    assert not g._rm.ready                      # nothing above needed the rows
    kbuf = g.kbuf                               # materialise
    ref = P.operators.DenseOperator.from_matrix(kbuf[:, :n].contiguous())
    full = D.empty(int(N.lib().dcg_packed_sym_doubles(n)))
    N.check(N.lib().dcg_pack_sym(D.ctx(), D.stream(), kbuf.data_ptr(), g.ldk, n, full.data_ptr()))
    assert torch.equal(full, g._packed.buf)
    assert torch.equal(ref.scaled(s, 1.0).matvec_dev(v), y_packed_only)
    assert torch.equal(ref.scaled(s, 1.0).apply_block_dev(w16), yb16)
    w24 = torch.from_numpy(rng.standard_normal((n, 24))).cuda()
    g2 = P.rbf_kernel(x, params)
    y24 = g2.scaled(s, 1.0).apply_block_dev(w24)   # k = 24: row-major product, materialised on demand
    assert g2._rm.ready
    assert torch.equal(y24, ref.scaled(s, 1.0).apply_block_dev(w24))


def test_packed_solve_early_exits(P):
    """The packed-tile solve's early exits with bulk copies of the next pass in
    flight (drained before the kernel returns): breakdown on an indefinite
    operator (solvers.py:170-172) and a zero right-hand side after a
    warm-start product (solvers.py:142-147), n = 4500 (symmetric strategy)."""
    import torch

    n = 4500
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.standard_normal((n, 6))).cuda()
    g = P.rbf_kernel(x, P.KernelParams(1.0, 1.4))
    assert g.c_struct().d_kp
    a = g.scaled(None, -0.5)            # K - 0.5 I: indefinite
    b = torch.from_numpy(rng.standard_normal(n)).cuda()
    with pytest.raises(P.BreakdownZeroCurvature):
        P.cg_solve(a, b, None, P.SolverConfig(tol=1e-10))
    spd = g.scaled(None, 1.0)
    w = torch.from_numpy(rng.standard_normal((n, 6))).cuda()
    basis = P.refresh_basis(spd, w)
    xs, rep, _ = P.deflated_cg_solve(spd, torch.zeros(n, dtype=torch.float64, device="cuda"),
                                     torch.from_numpy(rng.standard_normal(n)).cuda(), basis,
                                     P.SolverConfig(tol=1e-10, ell=8))
    assert rep.iterations == 0 and rep.residual_history == [0.0]
    assert not bool(torch.any(xs != 0))
    # and the library is still healthy afterwards
    xs, rep, _ = P.cg_solve(spd, b, None, P.SolverConfig(tol=1e-10))
    assert rep.converged


def test_packed_only_operator_with_offset_views(P):
    """Unaligned (offset) vector views handed to a packed-only operator (no
    row-major storage to fall back on) give the aligned results."""
    import torch

    n = 4500
    rng = np.random.default_rng(9)
    g = P.rbf_kernel(torch.from_numpy(rng.standard_normal((n, 5))).cuda(), P.KernelParams(1.0, 1.3))
    buf = torch.from_numpy(rng.standard_normal(n + 1)).cuda()
    v_off = buf[1:]                        # 8-byte offset
    assert v_off.data_ptr() % 16 == 8
    y1 = g @ v_off
    y2 = g @ v_off.clone()
    assert torch.equal(y1, y2)
    x, rep, _ = P.cg_solve(g.scaled(None, 1.0), v_off, None, P.SolverConfig(tol=1e-10))
    assert rep.converged
    assert not g._rm.ready
