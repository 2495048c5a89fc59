"""GPU: basis refresh, harmonic-Ritz extraction and solve_next against the
reference's known answers (pkg/tests/test_recycle.py) and its outputs on
identical inputs.  Eigenvector signs and rotations inside clusters are
rounding-dependent, so extracted bases are compared as SPANS (projectors),
Ritz values to 1e-9 relative, iteration counts to +-1."""

import numpy as np
import pytest

from conftest import golden, random_spd
from oracle import defcg_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1706_00241_b200 as P

    return P


def span_gap(u, v):
    qu, _ = np.linalg.qr(u)
    qv, _ = np.linalg.qr(v)
    return np.linalg.norm(qu @ qu.T - qv @ qv.T, 2)


def test_full_krylov_recovers_spectrum(P):
    _, _, log = P.cg_solve(np.diag([1.0, 2.0, 3.0]), np.ones(3), cfg=P.SolverConfig(tol=1e-14))
    assert log.stored_iterations == 3
    ext = P.harmonic_ritz_extract(log, None, 3)
    assert np.allclose(ext.theta, [1.0, 2.0, 3.0], atol=1e-8)


def test_k_zero_empty(P, rng):
    _, _, log = P.cg_solve(random_spd(rng, 6), rng.standard_normal(6), cfg=P.SolverConfig(tol=1e-12))
    ext = P.harmonic_ritz_extract(log, None, 0)
    assert ext.theta.shape == (0,) and ext.w_next.shape == (6, 0)


def test_early_convergence_uses_actual_count(P):
    a = np.diag([1.0, 2.0, 50.0, 60.0, 70.0])
    basis = P.refresh_basis(a, np.eye(5)[:, [0, 1]])
    _, rep, log = P.deflated_cg_solve(a, np.array([0.0, 0.0, 1.0, 1.0, 0.0]), np.zeros(5), basis,
                                      P.SolverConfig(tol=1e-10, ell=12))
    m = log.stored_iterations
    assert m == rep.iterations < 12
    ext = P.harmonic_ritz_extract(log, basis, 2)
    assert ext.z.shape[1] == basis.k + m


def test_selection_largest(P):
    _, _, log = P.cg_solve(np.diag([1.0, 2.0, 3.0, 4.0]), np.ones(4), cfg=P.SolverConfig(tol=1e-14))
    ext = P.harmonic_ritz_extract(log, None, 2, selection="largest")
    assert np.allclose(ext.theta, [3.0, 4.0], atol=1e-7)
    with pytest.raises(ValueError):
        P.harmonic_ritz_extract(log, None, 2, selection="middle")


def test_w_next_is_z_times_u(P, rng):
    _, _, log = P.cg_solve(random_spd(rng, 10), rng.standard_normal(10), cfg=P.SolverConfig(tol=1e-12))
    ext = P.harmonic_ritz_extract(log, None, 3)
    assert np.allclose(ext.w_next, ext.z @ ext.u, atol=1e-14)
    assert np.allclose(np.linalg.norm(ext.w_next, axis=0), 1.0, atol=1e-12)


def test_requested_k_too_large(P, rng):
    _, _, log = P.cg_solve(random_spd(rng, 6), rng.standard_normal(6), cfg=P.SolverConfig(tol=1e-12))
    with pytest.raises(P.BasisDeficient) as ei:
        P.harmonic_ritz_extract(log, None, log.stored_iterations + 1)
    assert ei.value.remaining == log.stored_iterations


def test_invariant_subspace(P):
    a = np.diag([1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    _, _, log = P.cg_solve(a, np.array([1.0, 1.0, 1.0, 0.0, 0.0, 0.0]), cfg=P.SolverConfig(tol=1e-13))
    ext = P.harmonic_ritz_extract(log, None, 3)
    assert np.allclose(ext.theta, [1.0, 2.0, 3.0], atol=1e-6)


def test_exact_invariant_subspace_with_prev_basis(P):
    a = np.diag([1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0])
    prev = P.refresh_basis(a, np.eye(7)[:, [0, 3]])
    b = np.zeros(7)
    b[[1, 4, 6]] = 1.0
    _, _, log = P.deflated_cg_solve(a, b, np.zeros(7), prev, P.SolverConfig(tol=1e-13))
    ext = P.harmonic_ritz_extract(log, prev, 5)
    assert np.allclose(np.sort(ext.theta), [1.0, 2.0, 4.0, 5.0, 7.0], atol=1e-6)


def test_pencil_residual(P, rng):
    a = random_spd(rng, 12, kappa=50.0)
    _, _, log = P.cg_solve(a, rng.standard_normal(12), cfg=P.SolverConfig(tol=1e-12, ell=8))
    ext = P.harmonic_ritz_extract(log, None, 4)
    az = a @ ext.z
    for theta, u in zip(ext.theta, ext.u.T):
        v = ext.z @ u
        res = az.T @ (a @ v - theta * v)
        assert np.linalg.norm(res) <= 1e-6 * np.linalg.norm(a @ v)


def test_ritz_parity_with_reference(P):
    g = golden("recycle_compiled")
    a, b = g["c_ritz_a"], g["c_ritz_b"]
    _, _, log = P.cg_solve(a, b, None, P.SolverConfig(tol=1e-10, ell=12))
    for sel in ("smallest", "largest"):
        ext = P.harmonic_ritz_extract(log, None, 5, sel)
        assert np.allclose(ext.theta, g[f"c_ritz_{sel}_theta"], rtol=1e-9)
        assert span_gap(ext.w_next, g[f"c_ritz_{sel}_w"]) < 1e-7
        assert np.allclose(np.abs(np.sum(ext.w_next * g[f"c_ritz_{sel}_w"], axis=0)), 1.0, atol=1e-7)


# ---------------------------------------------------------------- refresh
def test_refresh_single_column(P):
    basis = P.refresh_basis(np.diag([4.0, 5.0]), np.array([[1.0], [0.0]]))
    assert np.allclose(basis.aw, [[4.0], [0.0]], atol=1e-15)
    assert np.allclose(basis.gram_chol, [[2.0]], atol=1e-15)


def test_refresh_prunes_duplicates_like_reference(P, rng):
    g = golden("recycle_compiled")
    basis = P.refresh_basis(g["c_ritz_a"], g["c_refresh_w_in"])
    assert basis.k == 3
    assert np.array_equal(basis.w, g["c_refresh_w"])
    assert np.allclose(basis.aw, g["c_refresh_aw"], rtol=1e-12, atol=1e-12)
    assert np.allclose(basis.gram_chol, g["c_refresh_chol"], rtol=1e-12)
    w = rng.standard_normal((6, 1))
    assert P.refresh_basis(random_spd(rng, 6), np.hstack([w, w])).k == 1


def test_refresh_all_pruned_and_empty(P):
    with pytest.raises(P.BasisDeficient) as ei:
        P.refresh_basis(np.eye(3), np.zeros((3, 2)))
    assert ei.value.remaining == 0
    assert P.refresh_basis(np.eye(3), np.empty((3, 0))).k == 0


def test_refresh_eigenvector_basis(P, rng):
    a = random_spd(rng, 8)
    pairs = O.sym_eigen(a)
    basis = P.refresh_basis(a, pairs[1][:, :2])
    gram = basis.gram_chol @ basis.gram_chol.T
    assert np.allclose(gram, np.diag(pairs[0][:2]), atol=1e-10)


@pytest.mark.parametrize("n,k", [(9, 3), (1000, 16), (3001, 32), (700, 40)])
def test_refresh_aw_consistency(P, rng, n, k):
    """A.W on FP64 tensor cores vs an fp64 host product, including the implicit Newton operator."""
    a = random_spd(rng, n, 1e3) if n < 1200 else None
    if a is None:
        x = rng.standard_normal((n, 5))
        a = O.rbf_kernel(x, 1.0, 1.5)
    w = rng.standard_normal((n, k))
    basis = P.refresh_basis(a, w)
    ref = a @ w
    err = np.linalg.norm(basis.aw - ref, axis=0) / np.linalg.norm(ref, axis=0)
    assert basis.k == k and np.all(err <= 1e-12)
    # implicit A = I + S K S
    s = rng.uniform(0.1, 0.5, n)
    op = P.DenseOperator.from_matrix(a).scaled(s, 1.0)
    basis2 = P.refresh_basis(op, w)
    ref2 = (a * np.outer(s, s) + np.eye(n)) @ w
    err2 = np.linalg.norm(basis2.aw - ref2, axis=0) / np.linalg.norm(ref2, axis=0)
    assert np.all(err2 <= 1e-12)


# ---------------------------------------------------------------- solve_next
def test_first_solve_equals_plain_cg(P, rng):
    a = random_spd(rng, 12)
    b = rng.standard_normal(12)
    cfg = P.SolverConfig(tol=1e-10)
    x, st = P.solve_next(P.SequenceState(k=4, cfg=cfg), a, b)
    x_ref, rep_ref, _ = P.cg_solve(a, b, cfg=cfg)
    assert np.array_equal(x, x_ref)
    assert st.history[0].residual_history == rep_ref.residual_history
    assert st.basis is not None


def test_constant_sequence_recycling_helps(P):
    a = np.diag(np.arange(1.0, 41.0))
    st = P.SequenceState(k=5, cfg=P.SolverConfig(tol=1e-8, ell=10))
    _, st = P.solve_next(st, a, np.ones(40))
    _, st = P.solve_next(st, a, np.ones(40))
    assert st.history[1].iterations < st.history[0].iterations


def test_k_zero_always_plain_cg(P, rng):
    a = random_spd(rng, 15)
    b = rng.standard_normal(15)
    cfg = P.SolverConfig(tol=1e-9)
    st = P.SequenceState(k=0, cfg=cfg)
    _, st = P.solve_next(st, a, b)
    _, st = P.solve_next(st, a, b)
    x_ref, r1, _ = P.cg_solve(a, b, cfg=cfg)
    _, r2, _ = P.cg_solve(a, b, x0=x_ref, cfg=cfg)
    assert st.history[0].residual_history == r1.residual_history
    assert st.history[1].residual_history == r2.residual_history


def _permuted_reference_iterations(g, n_perm=32):
    """Iteration counts of the reference algorithm (oracle, numpy backend) on
    symmetrically permuted copies of the golden sequence.  P A P^T, P b is the
    same system, so the spread of these counts is the reference's own
    sensitivity to summation order (n = 64, ~240 CG iterations at kappa 1e4:
    far past n, where finite-precision CG counts are rounding-driven)."""
    from oracle import defcg_oracle as O

    out = []
    n = g["c_seq_b"].shape[1]
    for seed in range(n_perm):
        p = np.random.default_rng(seed).permutation(n)
        st = O.Sequence(k=4, cfg=O.Cfg(tol=1e-9, ell=10), selection="largest")
        its = []
        for i in range(4):
            _, st = O.solve_next(st, g["c_seq_a"][i][np.ix_(p, p)], g["c_seq_b"][i][p], be="numpy")
            its.append(st.history[-1].iterations)
        out.append(its)
    return np.array(out)


def test_sequence_parity_with_reference(P):
    """Iterations inside the reference's own rounding spread (compiled, numpy
    and 32 permuted-order runs, +-1); x within 1e-7 of the reference."""
    g, gn = golden("recycle_compiled"), golden("recycle_numpy")
    ens = _permuted_reference_iterations(g)
    st = P.SequenceState(k=4, cfg=P.SolverConfig(tol=1e-9, ell=10), selection="largest")
    for i in range(4):
        x, st = P.solve_next(st, g["c_seq_a"][i], g["c_seq_b"][i])
        ref, alt = int(g["c_seq_its"][i]), int(gn["n_seq_its"][i])
        lo = min(ref, alt, int(ens[:, i].min())) - 1
        hi = max(ref, alt, int(ens[:, i].max())) + 1
        assert lo <= st.history[-1].iterations <= hi, (i, st.history[-1].iterations, ref, lo, hi)
        xr = g["c_seq_x"][i]
        assert np.linalg.norm(x - xr) / np.linalg.norm(xr) <= 1e-7


def test_basis_deficient_degenerates_like_reference(P):
    """k larger than the first solve's logged iterations: BasisDeficient is
    swallowed and every later solve is plain CG (recycle.py:194-195)."""
    a = np.diag(np.arange(1.0, 11.0))
    cfg = P.SolverConfig(tol=1e-12, ell=3)
    st = P.SequenceState(k=5, cfg=cfg)
    _, st = P.solve_next(st, a, np.ones(10))
    assert st.basis is None
    x, st = P.solve_next(st, a, np.ones(10))
    assert st.basis is None and st.history[-1].iterations <= 1


def test_warm_start_carries_solution(P, rng):
    a = random_spd(rng, 10)
    b = rng.standard_normal(10)
    st = P.SequenceState(k=2, cfg=P.SolverConfig(tol=1e-10))
    _, st = P.solve_next(st, a, b)
    _, st = P.solve_next(st, a, b)
    assert st.history[1].iterations <= 1


def _set_pencil_fast(on):
    import ctypes

    from paper_1706_00241_b200 import _native as N

    fn = N.lib().dcg_debug_set_pencil_fast
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_int]
    assert fn(1 if on else 0) == 0


# well-conditioned pencils (cond F < 1e2): on a nearly singular F the two
# formations -- explicit C here, the one-sided X = L^-1 chol(G) there -- agree
# only to cond(F) eps
def _pencil_profile():
    import ctypes

    import torch

    from paper_1706_00241_b200 import _native as N

    torch.cuda.synchronize()
    h = (ctypes.c_longlong * 16)()
    N.lib().dcg_debug_pencil_profile.restype = ctypes.c_int
    assert N.lib().dcg_debug_pencil_profile(h) == 0
    return list(h)


@pytest.mark.parametrize("n,ell,k,kappa", [(60, 14, 4, 1e3), (120, 30, 8, 1e4), (200, 40, 16, 1e3), (300, 48, 16, 1e4),
                                           (500, 64, 32, 1e3)])
def test_pencil_tridiagonal_path_matches_jacobi(P, rng, n, ell, k, kappa):
    """The pencil's tridiagonal fast path (pencil_tridiag_fast) and the cyclic
    Jacobi path select the same Ritz pairs: values to 1e-9 relative, vectors as
    spans (both paths, both selections; T = ell stored directions >= 12)."""
    a = random_spd(rng, n, kappa=kappa)
    _, _, log = P.cg_solve(a, rng.standard_normal(n), cfg=P.SolverConfig(tol=1e-14, ell=ell))
    taken = 0
    try:
        for sel in ("smallest", "largest"):
            _set_pencil_fast(True)
            ef = P.harmonic_ritz_extract(log, None, k, sel)
            taken += _pencil_profile()[14]
            _set_pencil_fast(False)
            ej = P.harmonic_ritz_extract(log, None, k, sel)
            assert np.allclose(ef.theta, ej.theta, rtol=1e-9, atol=0)
            assert span_gap(ef.w_next, ej.w_next) < 1e-7
            assert np.allclose(np.linalg.norm(ef.w_next, axis=0), 1.0, atol=1e-12)
        assert taken >= 1   # the fast path ran (it may decline a clustered selection)
    finally:
        _set_pencil_fast(True)


def test_pencil_fast_path_declines_a_cluster(P):
    """A selected double eigenvalue (two exact eigenvectors of the same value
    carried in the previous basis): the tridiagonal fast path must decline
    (twisted-factorisation vectors of a cluster are not orthogonal) and the
    Jacobi path answers -- both copies of the value, their span exactly."""
    n = 80
    ev = np.arange(1.0, n + 1.0)
    ev[5] = ev[4]                      # eigenvalue 5 twice (coordinates 4 and 5)
    a = np.diag(ev)
    prev = P.refresh_basis(a, np.eye(n)[:, [4, 5]])
    rng = np.random.default_rng(3)
    b = rng.standard_normal(n)
    b[[4, 5]] = 0.0
    _, _, log = P.deflated_cg_solve(a, b, np.zeros(n), prev, P.SolverConfig(tol=1e-14, ell=16))
    assert prev.k + log.stored_iterations >= 12
    _set_pencil_fast(True)
    ext = P.harmonic_ritz_extract(log, prev, 6, "smallest")
    assert _pencil_profile()[14] == 0          # declined
    assert np.sum(np.abs(ext.theta - 5.0) < 1e-8) == 2
    e45 = np.eye(n)[:, [4, 5]]
    proj = ext.w_next @ np.linalg.pinv(ext.w_next)
    assert np.linalg.norm(proj @ e45 - e45) < 1e-8
