"""Report parity layer: the reference harness's output files from GPU runs.

A GPU Newton comparison written in the file formats of the reference's
experiment harness (/root/reference/pkg/src/defcg/bench.py: the record and
summary fields of `execute` :177-242, the three files of `emit_reports`
:276-333, delta = |value - ref| / |ref| :161-163), so a GPU run and a CPU run
can be diffed with the reference's own tooling: same columns, floats as
17 significant digits, summary keys sorted.  The subset-of-data baseline
(subset.py, run on the device) fills `subset` / `subset.csv` for each
requested fraction (bench.py:243-275).  Times are the GPU solve times of
NewtonRecord.solve_time_s.
"""

from __future__ import annotations

import csv
import json
from pathlib import Path

from . import _device as D
from .gpc import SOLVER_CHOLESKY, laplace_newton, rbf_kernel
from .solvers import SolverConfig

TABLE_COLUMNS = ("newton_iter", "solver", "logp", "rel_error_delta", "solver_iterations", "cumulative_time_s")
SUBSET_COLUMNS = ("fraction", "newton_iter", "cpu_time", "rel_logp_error")


def rel_error_delta(value, reference):
    """Relative deviation of a log-likelihood from the Cholesky solver's."""
    return abs(value - reference) / abs(reference)


def _solver_summary(recs):
    times = [r.solve_time_s for r in recs]
    its = [r.solver_iterations for r in recs]
    return {
        "newton_iterations": len(recs),
        "final_psi": float(recs[-1].psi),
        "final_loglik": float(recs[-1].loglik),
        "solver_iterations": its,
        "total_solver_iterations": sum(i or 0 for i in its),
        "total_solve_time_s": float(sum(times)),
        "residual_histories": [[float(h) for h in r.residual_history] for r in recs],
    }


def run_comparison(x, y, params, solvers=(SOLVER_CHOLESKY, "cg", "defcg"), solver_cfg: SolverConfig | None = None,
                   newton_tol=1.0, max_newton=30, k=8, selection="largest", jitter=None, config=None,
                   subset_fractions=(), seed=0):
    """One Laplace-Newton run per solver on the GPU.  Returns (rows, summary):
    rows are dicts keyed by TABLE_COLUMNS (plus `logp_tracked` = psi)."""
    solver_cfg = solver_cfg or SolverConfig()
    kernel = rbf_kernel(D.to_dev(x, 2), params, jitter)   # the Gram stays on the device for all solvers
    runs = {s: laplace_newton(kernel, y, solver=s, cfg=solver_cfg, newton_tol=newton_tol, max_newton=max_newton,
                              k=k, selection=selection)[1] for s in solvers}
    # the Cholesky run is the reference of the delta column (present when it ran first)
    ref_ll = [r.loglik for r in runs[SOLVER_CHOLESKY]] if SOLVER_CHOLESKY in runs else None
    rows = []
    for s in solvers:
        elapsed = 0.0
        for idx, r in enumerate(runs[s]):
            elapsed += r.solve_time_s
            earlier = ref_ll is not None and solvers.index(SOLVER_CHOLESKY) <= solvers.index(s)
            delta = rel_error_delta(r.loglik, ref_ll[idx]) if (earlier and idx < len(ref_ll)) else None
            rows.append({"newton_iter": r.newton_iter, "solver": s, "logp": r.loglik, "logp_tracked": r.psi,
                         "rel_error_delta": delta, "solver_iterations": r.solver_iterations,
                         "cumulative_time_s": elapsed})
    summary = {"config": dict(config or {}), "backend": "b200", "dataset_size": int(len(y)),
               "lengthscale_used": float(params.lengthscale), "subset": {},
               "solvers": {s: _solver_summary(recs) for s, recs in runs.items()}}
    if ref_ll is not None:
        summary["reference_final_loglik"] = float(ref_ll[-1])
        for s, recs in runs.items():
            summary["solvers"][s]["rel_error_to_final"] = [rel_error_delta(r.loglik, ref_ll[-1]) for r in recs]
    for frac in subset_fractions:
        # subset-of-data baseline (bench.py:243-275): cumulative subset solve
        # time against the full-data log-likelihood of the induced latents
        from .gpc import likelihood_derivs
        from .subset import assemble_full_latents, fit_subset

        model, recs = fit_subset(x, y, frac, params, newton_tol=newton_tol, seed=seed, jitter=jitter,
                                 max_newton=max_newton)
        elapsed, points = 0.0, []
        for r in recs:
            elapsed += r.solve_time_s
            loglik, _, _ = likelihood_derivs(assemble_full_latents(model, r.f), y)
            point = {"newton_iter": r.newton_iter, "cpu_time": elapsed, "loglik": float(loglik)}
            if ref_ll is not None:
                point["rel_logp_error"] = rel_error_delta(loglik, ref_ll[-1])
            points.append(point)
        summary["subset"][str(frac)] = {"m": model.m, "points": points}
    summary["complete"] = True
    return rows, summary


def _cell(v):
    if v is None:
        return ""
    return f"{v:.17g}" if isinstance(v, float) else str(v)


def _write_csv(path, columns, rows):
    with open(path, "w", encoding="utf-8", newline="") as fh:
        out = csv.writer(fh, lineterminator="\n")
        out.writerow(columns)
        out.writerows([[_cell(row.get(c)) for c in columns] for row in rows])


def emit_reports(rows, summary, output_path):
    """table.csv, summary.json, subset.csv under `output_path`."""
    out = Path(output_path)
    out.mkdir(parents=True, exist_ok=True)
    _write_csv(out / "table.csv", TABLE_COLUMNS, rows)
    (out / "summary.json").write_text(json.dumps(summary, indent=2, sort_keys=True) + "\n", encoding="utf-8")
    subset_rows = [{"fraction": frac, "newton_iter": p["newton_iter"], "cpu_time": p["cpu_time"],
                    "rel_logp_error": p.get("rel_logp_error")}
                   for frac, info in summary.get("subset", {}).items() for p in info["points"]]
    _write_csv(out / "subset.csv", SUBSET_COLUMNS, subset_rows)
