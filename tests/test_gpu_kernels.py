"""GPU: the L0 device twins of the reference kernel backend (_core.pyx) and
the L1 dense linear algebra, against the golden vectors the reference itself
produced (tests/golden/kernels_compiled.npz) and the oracle.

Tolerances: kernels that keep the reference's serial operation order with
non-contracted fp64 (Cholesky, triangular solves, i-k-j gemm, cyclic Jacobi)
must be BIT-IDENTICAL; reductions reordered for the GPU (GEMV rows) are
held to 4 ulp-scale relative error; the RBF Gram to 2 ulp (CUDA exp vs libm)."""

import numpy as np
import pytest

from conftest import golden, random_spd
from oracle import defcg_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1706_00241_b200 as P

    return P


@pytest.fixture(scope="module")
def g():
    return golden("kernels_compiled")


def test_matvec(P, g):
    y = P.matvec(g["c_mv_a"], g["c_mv_x"])
    ref = g["c_mv_y"]
    scale = np.abs(g["c_mv_a"]) @ np.abs(g["c_mv_x"])
    assert np.all(np.abs(y - ref) <= 8 * np.finfo(float).eps * scale)


def test_matvec_repeat_bit_identical(P, rng):
    a = rng.standard_normal((513, 1001))
    x = rng.standard_normal(1001)
    y1, y2 = P.matvec(a, x), P.matvec(a, x)
    assert np.array_equal(y1, y2)


def test_gemm_bitwise(P, g):
    assert np.array_equal(P.gemm(g["c_mv_a"], g["c_gemm_b"]), g["c_gemm_c"])


def test_cholesky_bitwise(P, g):
    low = P.cholesky_factor(g["c_chol_a"])
    assert np.array_equal(low, g["c_chol_l"])


def test_cholesky_failure_index(P):
    with pytest.raises(P.NotPositiveDefinite) as ei:
        P.cholesky_factor(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert ei.value.pivot_index == 1
    assert np.array_equal(P.cholesky_factor(np.array([[4.0, 2.0], [2.0, 5.0]])), [[2.0, 0.0], [1.0, 2.0]])


def test_triangular_solves_bitwise(P, g):
    from paper_1706_00241_b200 import linalg

    low = g["c_chol_l"]
    assert np.array_equal(linalg.solve_lower(low, g["c_sl_b"]), g["c_sl_y"])
    assert np.array_equal(linalg.solve_lower_trans(low, g["c_sl_b"]), g["c_slt_x"])


def test_rbf_gram(P, g):
    from paper_1706_00241_b200 import kernels

    x = g["c_rbf_x"]
    k = kernels.rbf_gram(x, 1.7, 1.0 / (2 * 1.3**2), 1e-3)
    ref = g["c_rbf_k"]
    assert np.array_equal(k, k.T)                       # exact symmetry by construction
    assert np.array_equal(np.diag(k), np.full(len(x), 1.7 + 1e-3))   # exact diagonal
    assert np.max(np.abs(k - ref) / np.abs(ref)) <= 4 * np.finfo(float).eps


def test_jacobi_sweep_bitwise(P, g):
    from paper_1706_00241_b200 import linalg

    a = g["c_jac_a"].copy()
    v = np.eye(a.shape[0])
    rot = linalg.jacobi_sweep(a, v)
    assert rot == int(g["c_jac_rot"])
    assert np.array_equal(a, g["c_jac_a1"]) and np.array_equal(v, g["c_jac_v1"])


def test_sym_eigen_matches_oracle(P, rng):
    for n in (1, 2, 7, 30, 68):
        a = random_spd(rng, n, 1e3) - 3.0 * np.eye(n)
        pairs = P.sym_eigen(a)
        vals, vecs = O.sym_eigen(a)
        assert np.allclose(pairs.values, vals, rtol=1e-12, atol=1e-12 * np.abs(vals).max())
        # same eigenvectors up to sign (spectrum is simple here)
        dots = np.abs(np.sum(pairs.vectors * vecs, axis=0))
        assert np.allclose(dots, 1.0, atol=1e-9)
        assert np.allclose(pairs.vectors.T @ pairs.vectors, np.eye(n), atol=1e-12)


def test_sym_eigen_zero_and_diagonal(P):
    z = P.sym_eigen(np.zeros((4, 4)))
    assert np.array_equal(z.values, np.zeros(4)) and np.array_equal(z.vectors, np.eye(4))
    d = P.sym_eigen(np.diag([3.0, 1.0, 2.0]))
    assert np.array_equal(d.values, [1.0, 2.0, 3.0])


def test_gen_sym_eigen(P, rng):
    for n in (3, 12, 40):
        g_ = random_spd(rng, n, 50.0)
        f_ = random_spd(rng, n, 10.0)
        pairs = P.gen_sym_eigen(g_, f_)
        vals, vecs = O.gen_sym_eigen(g_, f_)
        assert np.allclose(pairs.values, vals, rtol=1e-11)
        for j in range(n):
            u = pairs.vectors[:, j]
            res = g_ @ u - pairs.values[j] * (f_ @ u)
            assert np.linalg.norm(res) <= 1e-9 * np.abs(g_).max() * np.sqrt(n)
            assert abs(np.linalg.norm(u) - 1.0) < 1e-12
    with pytest.raises(P.NotPositiveDefinite):
        P.gen_sym_eigen(np.eye(2), np.array([[1.0, 2.0], [2.0, 1.0]]))


def test_require_symmetric(P):
    from paper_1706_00241_b200 import linalg

    a = np.array([[1.0, 2.0], [2.0 + 1e-13, 1.0]])
    linalg.require_symmetric(a)
    with pytest.raises(ValueError):
        linalg.require_symmetric(np.array([[1.0, 2.0], [2.1, 1.0]]))
    with pytest.raises(P.DimensionMismatch):
        linalg.require_symmetric(np.ones((2, 3)))
    big = random_spd(np.random.default_rng(3), 300)
    big[7, 250] += 1e-6
    with pytest.raises(ValueError):
        linalg.require_symmetric(big)


def test_raw_matrix_never_mutated(P, rng):
    """A torch fp64 CUDA input whose row pitch needs no padding (n % 32 == 0)
    is used in place by the operator: it must come back bit-identical, also
    when it is symmetric only within the tolerance (that operator then streams
    full rows, the reference's own matvec)."""
    import torch

    n = 1024
    a = rng.standard_normal((n, n))
    a = a @ a.T / n + np.eye(n)
    a_pert = a + np.triu(1e-15 * rng.standard_normal((n, n)), 1)     # asymmetric within 1e-12 max|A|
    for mat in (a, a_pert):
        t = torch.from_numpy(mat.copy()).cuda()
        before = t.clone()
        b = rng.standard_normal(n)
        x, rep, _ = P.cg_solve(t, torch.from_numpy(b).cuda(), None, P.SolverConfig(tol=1e-10))
        assert torch.equal(t, before)
        xo, repo, _ = O.cg_solve(mat, b, None, O.Cfg(tol=1e-10))
        assert abs(rep.iterations - repo.iterations) <= 1
        assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-8 * np.linalg.norm(xo)
    op = P.operators.DenseOperator.from_matrix(torch.from_numpy(a_pert).cuda())
    assert op.strategy == "rows"
    assert P.operators.DenseOperator.from_matrix(torch.from_numpy(a).cuda()).strategy != "rows"
