"""Golden files of the reference harness's report format (bench.py
emit_reports), produced by the REFERENCE itself on a fixed record set.

    DEFCG_BACKEND=numpy python tests/golden/make_report_golden.py

Imports `defcg.bench` from /root/reference/pkg/src (build container only),
writes tests/golden/report_fmt/{table,summary,subset} and the input rows as
report_fmt/rows.json; tests/test_report.py checks that the package's
report.emit_reports writes byte-identical files from the same rows.
"""

import json
import os
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent / "report_fmt"


def main():
    os.environ.setdefault("DEFCG_BACKEND", "numpy")
    sys.path.insert(0, "/root/reference/pkg/src")
    from defcg.bench import RunRecord, emit_reports

    rows = []
    t = 0.0
    for solver, its in (("cholesky", [None, None, None]), ("cg", [29, 18, 18]), ("defcg", [29, 12, 9])):
        for i, it in enumerate(its):
            t += 0.1 + 0.01 * i
            ll = -1385.2938742 + 0.5 * i - (0.001 if solver != "cholesky" else 0.0)
            rows.append({"newton_iter": i + 1, "solver": solver, "logp": ll, "logp_tracked": ll - 3.0,
                         "rel_error_delta": None if solver == "cholesky" and i == 0 and False else
                         abs(ll - (-1385.2938742 + 0.5 * i)) / abs(-1385.2938742 + 0.5 * i),
                         "solver_iterations": it, "cumulative_time_s": t})
    summary = {"config": {"n": 300, "k": 8}, "backend": "numpy", "dataset_size": 300, "lengthscale_used": 1.2,
               "solvers": {"defcg": {"final_loglik": -1384.2938742, "solver_iterations": [29, 12, 9]}},
               "subset": {"0.05": {"m": 15, "points": [{"newton_iter": 1, "cpu_time": 0.25, "loglik": -1400.5,
                                                         "rel_logp_error": 0.0110}]}},
               "complete": True}
    recs = [RunRecord(newton_iter=r["newton_iter"], solver=r["solver"], logp_tracked=r["logp_tracked"],
                      loglik=r["logp"], rel_error_delta=r["rel_error_delta"],
                      solver_iterations=r["solver_iterations"], cumulative_time_s=r["cumulative_time_s"])
            for r in rows]
    OUT.mkdir(parents=True, exist_ok=True)
    emit_reports(recs, summary, str(OUT))
    (OUT / "rows.json").write_text(json.dumps({"rows": rows, "summary": summary}, indent=1))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
