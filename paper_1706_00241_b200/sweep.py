"""GP-regression hyperparameter sweep with a recycled deflation basis.

The reference has no driver for this workload; it is
composed strictly from the reference's public API, one system per
lengthscale theta:

    A_theta = rbf_kernel(X, KernelParams(signal_sd, theta), jitter=sigma2)   gpc.py:82-98
    x_theta, state = solve_next(state, A_theta, y)                          recycle.py:162-203

On the device the Gram matrix of each theta is assembled in HBM (K6) into a
buffer reused across thetas, and W / AW / x_last never leave the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from .gpc import KernelParams, rbf_kernel
from .recycle import SELECT_LARGEST, SequenceState, solve_next
from .solvers import SolveReport, SolverConfig


@dataclass
class SweepRecord:
    theta: float
    iterations: int
    rel_residual: float
    solve_time_s: float
    report: SolveReport


def hyperparameter_sweep(x, y, lengthscales, signal_sd=1.0, jitter=0.01, k=24, cfg=None,
                         selection=SELECT_LARGEST):
    """Solve (K_theta + jitter I) x = y for every lengthscale in order.

    Returns (list of solutions, list of SweepRecord); solutions are numpy
    arrays when ``y`` is a numpy array."""
    cfg = cfg or SolverConfig(tol=1e-8, ell=k + 4)
    xd = D.to_dev(x, 2)
    host = not isinstance(y, torch.Tensor)
    yd = D.to_dev(y, 1)
    state = SequenceState(k=k, cfg=cfg, selection=selection)
    sols, recs = [], []
    for theta in lengthscales:
        op = rbf_kernel(xd, KernelParams(signal_sd, float(theta)), jitter=jitter)
        xs, state = solve_next(state, op, yd, defer_extraction=True)
        rep = state.history[-1]
        recs.append(SweepRecord(float(theta), rep.iterations, rep.residual_history[-1], rep.wall_time, rep))
        sols.append(xs)
        del op
    _ = state.basis   # join the last pending extraction
    if host:
        sols = [s.cpu().numpy() for s in sols]
    return sols, recs


def default_lengthscales(count=20, lo=0.5, hi=2.0):
    """BASELINE config 4: 20 lengthscales log-spaced in [0.5, 2], ascending."""
    return np.logspace(np.log10(lo), np.log10(hi), count)
