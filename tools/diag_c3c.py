"""Second Newton solve of the config-3 recipe (n = 24k, permutation j of the
parity test) with the same recycled basis under each product strategy."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200 import gpc as G  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402

n = 24000
perm_no = int(sys.argv[1]) if len(sys.argv) > 1 else 4
x, y = gpc_inputs(n, 8)
if perm_no:
    rng = np.random.default_rng(12345)
    perm = [rng.permutation(n) for _ in range(perm_no)][-1]
    x, y = x[perm], y[perm]
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 2.0)).with_strategy("rows")
cfg = P.SolverConfig(tol=1e-8, ell=36)
st0 = G.make_state(gram, torch.from_numpy(y).cuda())
s1 = G.build_newton_system(st0)
seq = P.SequenceState(k=32, cfg=cfg, selection="largest")
x1, seq = P.solve_next(seq, s1.a_matrix, s1.b)
st1, psi1 = G._update_dev(st0, s1.inner, s1.sqrt_h, x1)
s2 = G.build_newton_system(st1)
basis = seq.basis
print("step1 its", seq.history[-1].iterations, "psi", psi1, "basis k", None if basis is None else basis.k)
for strat in ("rows", "sym_rowmajor", "sym"):
    A = s2.a_matrix.with_strategy(strat)
    x2, s_ = P.solve_next(seq, A, s2.b)
    rep = s_.history[-1]
    true = float(torch.linalg.norm(s2.b - s2.a_matrix.with_strategy("rows").matvec_dev(x2)) / torch.linalg.norm(s2.b))
    h = rep.residual_history
    print(strat, "its", rep.iterations, "rel", h[-1], "true", true, "hist", [f"{v:.2e}" for v in h[:8]], "...",
          [f"{v:.2e}" for v in h[-4:]])
