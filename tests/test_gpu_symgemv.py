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
