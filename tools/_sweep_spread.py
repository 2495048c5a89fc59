import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1706_00241_b200 as P
from oracle import defcg_oracle as O
from test_gpu_recycle import _set_pencil_fast
n, k = 700, 8
x, y = O.sweep_inputs(n, d=8, seed=0)
thetas = np.logspace(np.log10(0.5), np.log10(2.0), 6)
for fast in (1, 0):
    _set_pencil_fast(fast)
    for s in [None] + list(range(6)):
        perm = np.arange(n) if s is None else np.random.default_rng(s).permutation(n)
        _, recs = P.hyperparameter_sweep(x[perm], y[perm], thetas, k=k, cfg=P.SolverConfig(tol=1e-8, ell=k + 4))
        print("fast", fast, "perm", s, [r.iterations for r in recs])
