"""GPU: the report parity layer on a small GPC comparison -- every solver's
rows, the delta column against the GPU Cholesky run, and the reference's
summary schema."""

import numpy as np
import pytest

from oracle import defcg_oracle as O

pytestmark = pytest.mark.gpu


def test_run_comparison_rows_and_schema(tmp_path):
    import paper_1706_00241_b200 as P
    from paper_1706_00241_b200 import report

    x, y = O.gpc_inputs(300, 4, 0)
    rows, summary = report.run_comparison(x, y, P.KernelParams(1.0, 1.2), ("cholesky", "cg", "defcg"),
                                          P.SolverConfig(tol=1e-8, ell=8), newton_tol=-np.inf, max_newton=4, k=4)
    assert [r["solver"] for r in rows] == ["cholesky"] * 4 + ["cg"] * 4 + ["defcg"] * 4
    assert all(r["rel_error_delta"] is not None for r in rows)
    assert max(r["rel_error_delta"] for r in rows) <= 1e-7          # tol 1e-8 solves track the direct solve
    assert all(r["solver_iterations"] is None for r in rows[:4])
    assert set(summary) >= {"config", "backend", "dataset_size", "lengthscale_used", "solvers", "subset",
                            "reference_final_loglik", "complete"}
    assert set(summary["solvers"]["defcg"]) == {"newton_iterations", "final_psi", "final_loglik",
                                                "solver_iterations", "total_solver_iterations",
                                                "total_solve_time_s", "residual_histories", "rel_error_to_final"}
    report.emit_reports(rows, summary, tmp_path)
    lines = (tmp_path / "table.csv").read_text().splitlines()
    assert lines[0] == ",".join(report.TABLE_COLUMNS) and len(lines) == 13
