"""GPU: the subset-of-data baseline (subset.py:38-98) against
the oracle's Cholesky Newton fit of the same subset and a numpy restatement
of the induced latents."""

import numpy as np
import pytest

from oracle import defcg_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1706_00241_b200 as P

    return P


@pytest.mark.parametrize("frac", [0.05, 0.25, 1.0])
def test_fit_subset_matches_oracle(P, frac):
    x, y = O.gpc_inputs(1200, 5)
    params = P.KernelParams(2.0, 1.5)
    model, recs = P.fit_subset(x, y, frac, params, newton_tol=1e-9, seed=3)
    m = min(1200, max(1, int(round(frac * 1200))))
    idx = np.random.default_rng(3).choice(1200, size=m, replace=False)
    assert np.array_equal(model.indices_m, idx)
    _, _, ref = O.laplace_newton(O.rbf_kernel(x[idx], 2.0, 1.5), y[idx], "cholesky", newton_tol=1e-9)
    assert len(recs) == len(ref)
    for a, b in zip(recs, ref):
        assert abs(a.psi - b.psi) <= 1e-11 * abs(b.psi)
        assert np.linalg.norm(a.f - b.f) <= 1e-10 * max(np.linalg.norm(b.f), 1e-300)
    # induced latents: K_rest,m K_mm^-1 f_m (numpy restatement)
    f = P.assemble_full_latents(model)
    k_mm = O.rbf_kernel(x[idx], 2.0, 1.5)
    rest = np.setdiff1d(np.arange(1200), idx)
    if rest.size:
        d2 = ((x[rest][:, None, :] - x[idx][None, :, :]) ** 2).sum(-1)
        cross = 4.0 * np.exp(-d2 / (2 * 1.5**2))
        want = cross @ np.linalg.solve(k_mm, model.f_m)
        assert np.allclose(f[rest], want, rtol=1e-9, atol=1e-12)
    assert np.array_equal(f[idx], model.f_m)
    ll_full = P.evaluate_full(model, x, y)
    assert np.isfinite(ll_full)


def test_report_subset_rows(P, tmp_path):
    x, y = O.gpc_inputs(400, 4)
    rows, summary = P.report.run_comparison(x, y, P.KernelParams(2.0, 1.2), newton_tol=1e-6,
                                            subset_fractions=(0.1, 0.5), seed=1)
    assert set(summary["subset"]) == {"0.1", "0.5"}
    for info in summary["subset"].values():
        assert info["points"] and all("rel_logp_error" in p for p in info["points"])
    P.report.emit_reports(rows, summary, tmp_path)
    lines = (tmp_path / "subset.csv").read_text().splitlines()
    assert lines[0] == "fraction,newton_iter,cpu_time,rel_logp_error" and len(lines) > 2
