"""Conformance shim: the reference's synthetic two-cluster generator
(data.py:71-87), restated for the acceptance criteria's inputs."""
import numpy as np

from paper_1706_00241_b200.errors import DataError


def gen_synthetic(n, d, seed, separation):
    if n < 2:
        raise DataError(f"n must be at least 2, got {n}")
    if d < 1:
        raise DataError(f"d must be at least 1, got {d}")
    rng = np.random.default_rng(seed)
    n_pos = (n + 1) // 2
    x = rng.standard_normal((n, d))
    x[:n_pos, 0] += separation / 2.0
    x[n_pos:, 0] -= separation / 2.0
    y = np.concatenate([np.ones(n_pos, dtype=np.int64), -np.ones(n - n_pos, dtype=np.int64)])
    return x, y
