#!/usr/bin/env python
"""Config-1 comparison in the reference harness's report format, twice:
from the GPU path (paper_1706_00241_b200.report.run_comparison) and from the
CPU restatement of the reference (oracle, numpy backend), into

    profiles/r01_report_config1_gpu/{table.csv,summary.json,subset.csv}
    profiles/r01_report_config1_cpu/...

so the two can be diffed with the reference's own tooling.  Prints the
largest per-row differences (logp relative, solver iterations).

  python tools/report_config.py [out_root]
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import paper_1706_00241_b200 as P
    from oracle import defcg_oracle as O
    from paper_1706_00241_b200 import report

    out = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles"
    n, d, ell, k = 2000, 5, 1.5, 8
    x, y = O.gpc_inputs(n, d, 0)
    cfg_dict = {"n": n, "d": d, "lengthscale": ell, "k": k, "ell": k + 4, "tol": 1e-8, "newton_tol": "-inf",
                "max_newton": 8, "selection": "largest", "seed": 0}
    solvers = ("cholesky", "cg", "defcg")
    rows, summary = report.run_comparison(x, y, P.KernelParams(1.0, ell), solvers,
                                          P.SolverConfig(tol=1e-8, ell=k + 4), newton_tol=-np.inf, max_newton=8,
                                          k=k, selection="largest", config=cfg_dict)
    report.emit_reports(rows, summary, out / "r01_report_config1_gpu")

    # the same comparison through the oracle (CPU), same assembly
    kmat = O.rbf_kernel(x, 1.0, ell, be="numpy")
    runs = {s: O.laplace_newton(kmat, y, s, O.Cfg(tol=1e-8, ell=k + 4), newton_tol=-np.inf, max_newton=8, k=k,
                                selection="largest", be="numpy")[2] for s in solvers}
    ref_ll = [r.loglik for r in runs["cholesky"]]
    crow = []
    for s in solvers:
        t = 0.0
        for i, r in enumerate(runs[s]):
            t += r.solve_time_s
            crow.append({"newton_iter": r.newton_iter, "solver": s, "logp": r.loglik,
                         "rel_error_delta": report.rel_error_delta(r.loglik, ref_ll[i]) if i < len(ref_ll) else None,
                         "solver_iterations": r.solver_iterations, "cumulative_time_s": t})
    csum = {"config": cfg_dict, "backend": "oracle-numpy", "dataset_size": n, "lengthscale_used": ell, "subset": {},
            "solvers": {s: {"solver_iterations": [r.solver_iterations for r in recs],
                            "final_loglik": float(recs[-1].loglik)} for s, recs in runs.items()},
            "reference_final_loglik": float(ref_ll[-1]), "complete": True}
    report.emit_reports(crow, csum, out / "r01_report_config1_cpu")

    dl = max(abs(a["logp"] - b["logp"]) / abs(b["logp"]) for a, b in zip(rows, crow))
    di = max(abs((a["solver_iterations"] or 0) - (b["solver_iterations"] or 0)) for a, b in zip(rows, crow))
    print(json.dumps({"rows": len(rows), "max_rel_logp_diff": dl, "max_solver_iteration_diff": di,
                      "gpu_defcg_iterations": summary["solvers"]["defcg"]["solver_iterations"],
                      "cpu_defcg_iterations": csum["solvers"]["defcg"]["solver_iterations"]}))


if __name__ == "__main__":
    main()
