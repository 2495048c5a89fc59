"""Conformance shim: the reference harness's interface (bench.py:49-135,
161-163, 278-333) over paper_1706_00241_b200.report (GPU runs, the reference's
file formats)."""
from dataclasses import asdict, dataclass

from paper_1706_00241_b200 import report as _report
from paper_1706_00241_b200.errors import ConfigError
from paper_1706_00241_b200.gpc import KernelParams
from paper_1706_00241_b200.recycle import SELECT_LARGEST
from paper_1706_00241_b200.solvers import SolverConfig

from .data import gen_synthetic

ALL_SOLVERS = ("cholesky", "cg", "defcg")
rel_error_delta = _report.rel_error_delta


@dataclass
class ExperimentConfig:
    dataset: str = "synthetic"
    n: int = 2000
    d: int = 3
    separation: float = 3.0
    images_path: str | None = None
    labels_path: str | None = None
    digit_a: int = 3
    digit_b: int = 5
    max_n: int = 2000
    theta: float = 1.0
    lengthscale: float | None = None
    jitter: float | None = None
    tol: float = 1e-5
    max_iters: int | None = None
    ell: int = 12
    recompute_residual_every: int = 50
    k: int = 8
    selection: str = SELECT_LARGEST
    solvers: tuple = ALL_SOLVERS
    newton_tol: float = 1.0
    max_newton: int = 30
    subset_fractions: tuple = (0.05, 0.25)
    output_path: str = "results"
    seed: int = 0


@dataclass
class RunRecord:
    newton_iter: int
    solver: str
    logp_tracked: float
    loglik: float
    rel_error_delta: float | None
    solver_iterations: int | None
    cumulative_time_s: float


def run_comparison(cfg):
    if cfg.dataset != "synthetic":
        raise ConfigError("the conformance shim runs the synthetic dataset only")
    x, y = gen_synthetic(cfg.n, cfg.d, cfg.seed, cfg.separation)
    if cfg.lengthscale is None:
        raise ConfigError("the conformance shim needs an explicit lengthscale")
    params = KernelParams(signal_sd=cfg.theta, lengthscale=cfg.lengthscale)
    scfg = SolverConfig(tol=cfg.tol, max_iters=cfg.max_iters, ell=cfg.ell,
                        recompute_residual_every=cfg.recompute_residual_every)
    rows, summary = _report.run_comparison(x, y, params, solvers=tuple(cfg.solvers), solver_cfg=scfg,
                                           newton_tol=cfg.newton_tol, max_newton=cfg.max_newton, k=cfg.k,
                                           selection=cfg.selection, jitter=cfg.jitter, config=asdict(cfg),
                                           subset_fractions=tuple(cfg.subset_fractions), seed=cfg.seed)
    records = [RunRecord(r["newton_iter"], r["solver"], r["logp_tracked"], r["logp"], r["rel_error_delta"],
                         r["solver_iterations"], r["cumulative_time_s"]) for r in rows]
    return records, summary


def emit_reports(records, summary, output_path):
    rows = [{"newton_iter": r.newton_iter, "solver": r.solver, "logp": r.loglik, "rel_error_delta": r.rel_error_delta,
             "solver_iterations": r.solver_iterations, "cumulative_time_s": r.cumulative_time_s} for r in records]
    _report.emit_reports(rows, summary, output_path)
