"""Seeded synthetic inputs of the BASELINE.json configurations.

The reference's own workload (infinite-MNIST 3-vs-5) is not available; every
config is synthetic.  Inputs are drawn in numpy fp64 with
``default_rng(seed)``, X first and then the noise vector, so the same arrays go
to the GPU path, the oracle and the reference run that produced the goldens
(``tests/golden/make_golden*.py`` restate the same recipes).

Each GPC config is a Laplace-Newton sequence
``laplace_newton(rbf_kernel(X, KernelParams(1, lengthscale)), y, "defcg",
SolverConfig(tol, ell=k + 4), newton_tol=-inf, max_newton=8, k, "largest")``
(gpc.py:212-291); config 4 is the GP-regression sweep of §3.5.
"""

from __future__ import annotations

import numpy as np

CONFIGS = {
    1: dict(kind="gpc", n=2_000, d=5, lengthscale=1.5, k=8, ell=12, tol=1e-8, newton_steps=8),
    2: dict(kind="gpc", n=10_000, d=10, lengthscale=1.5, k=16, ell=20, tol=1e-8, newton_steps=8),
    3: dict(kind="gpc", n=50_000, d=8, lengthscale=2.0, k=32, ell=36, tol=1e-8, newton_steps=8),
    4: dict(kind="sweep", n=30_000, d=8, k=24, ell=28, tol=1e-8, thetas=20, jitter=0.01),
    5: dict(kind="gpc", n=200_000, d=16, lengthscale=3.0, k=32, ell=36, tol=1e-8, newton_steps=8,
            matrix_free=True),
}


def gpc_inputs(n, d, seed=0):
    """X ~ N(0, I_d) drawn first, then noise; y = sign(sum_j sin(2 x_j) + 0.1 noise), sign(0) -> +1."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d))
    noise = rng.standard_normal(n)
    t = np.sin(2.0 * x).sum(axis=1) + 0.1 * noise
    return x, np.where(t >= 0.0, 1.0, -1.0)


def sweep_inputs(n, d=8, seed=0):
    """Config 4: X ~ U[-1,1]^d, y = sum_j sin(3 x_j) + 0.05 noise (real-valued)."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1.0, 1.0, (n, d))
    noise = rng.standard_normal(n)
    return x, np.sin(3.0 * x).sum(axis=1) + 0.05 * noise


def sweep_thetas(count=20):
    """The 20 lengthscales log-spaced in [0.5, 2], ascending."""
    return np.logspace(np.log10(0.5), np.log10(2.0), count)
