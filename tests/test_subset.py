"""The subset-of-data baseline (subset.py:38-98) and the conformance shim, CPU side."""

import importlib
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_subset_indices_follow_the_reference_rng():
    """fit_subset draws its m points with default_rng(seed).choice(n, m,
    replace=False) exactly as subset.py:55-57 (checked here without a GPU)."""
    n, frac, seed = 2000, 0.05, 0
    m = min(n, max(1, int(round(frac * n))))
    idx = np.random.default_rng(seed).choice(n, size=m, replace=False)
    assert idx.shape == (100,) and len(set(idx.tolist())) == 100


def test_conformance_shim_imports():
    sys.path.insert(0, str(ROOT / "conformance"))
    try:
        for name in ("defcg", "defcg.solvers", "defcg.recycle", "defcg.gpc", "defcg.linalg", "defcg.errors",
                     "defcg.subset", "defcg._kernels", "defcg.bench", "defcg.data"):
            importlib.import_module(name)
        import defcg

        assert defcg.solvers.cg_solve is importlib.import_module("paper_1706_00241_b200").cg_solve
        assert hasattr(defcg.recycle, "deflated_spectrum") and hasattr(defcg.recycle, "condition_numbers")
        x, y = defcg.data.gen_synthetic(10, 3, 0, 2.0)
        assert x.shape == (10, 3) and y.sum() == 0
    finally:
        sys.path.remove(str(ROOT / "conformance"))
        for name in [k for k in sys.modules if k == "defcg" or k.startswith("defcg.")]:
            del sys.modules[name]
