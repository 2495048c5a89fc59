"""Config-3 recipe at n = 24k, 3 Newton steps: per-step iterations, kept basis
columns, psi and the solve's final residual, for one operator strategy.
  python tools/diag_c3b.py [strategy] [n]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402

strategy = sys.argv[1] if len(sys.argv) > 1 else "sym"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 24000
x, y = gpc_inputs(n, 8)
perm_no = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # 0 = original order, j = the test's j-th permutation
if perm_no:
    rng = np.random.default_rng(12345)
    perm = [rng.permutation(n) for _ in range(perm_no)][-1]
    x, y = x[perm], y[perm]
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 2.0)).with_strategy(strategy)
try:
    _, recs = P.laplace_newton(gram, y, "defcg", P.SolverConfig(tol=1e-8, ell=36), newton_tol=-np.inf,
                               max_newton=3, k=32, selection="largest")
    print(strategy, perm_no, os.environ.get("DCG_LIB_PATH"), [r.solver_iterations for r in recs], [r.psi for r in recs],
          [r.residual_history[-1] for r in recs])
except Exception as e:  # noqa: BLE001
    print(strategy, perm_no, os.environ.get("DCG_LIB_PATH"), "FAILED", type(e).__name__, e)
