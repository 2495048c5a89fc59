"""Our own rounding spread at a config recipe: the first Newton steps on
symmetric row permutations of the same data (as tests/golden/make_golden_big.py
does for the reference).  python tools/diag_perm.py n d lengthscale k steps nperm [matrix_free]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
n, d, ell, k, steps, nperm = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]),
                              int(sys.argv[5]), int(sys.argv[6]))
mf = len(sys.argv) > 7 and sys.argv[7] == "mf"
x, y = gpc_inputs(n, d)
rng = np.random.default_rng(12345)
perms = [None] + [rng.permutation(n) for _ in range(nperm)]
for perm in perms:
    xs, ys = (x, y) if perm is None else (x[perm], y[perm])
    gram = P.rbf_kernel(xs, P.KernelParams(1.0, ell), matrix_free=mf)
    _, recs = P.laplace_newton(gram, ys, "defcg", P.SolverConfig(tol=1e-8, ell=k + 4), newton_tol=-np.inf,
                               max_newton=steps, k=k, selection="largest")
    print("perm" if perm is not None else "orig", [r.solver_iterations for r in recs], flush=True)
    del gram
