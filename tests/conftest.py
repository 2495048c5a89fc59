"""Shared fixtures.  GPU tests are marked ``gpu``; everything else runs on CPU."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libdefcg_b200.so")


def random_spd(rng, n, kappa=100.0):
    """QR-based SPD matrix with eigenvalues log-spaced in [1, kappa] (the reference suite's construction)."""
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    a = q @ np.diag(np.logspace(0.0, np.log10(kappa), n)) @ q.T
    return 0.5 * (a + a.T)


def golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
