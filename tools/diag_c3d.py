"""Pipelined config-3 recipe Newton sequence (n = 24k, permutation j), the
NoProgress check disabled: per-step iterations and residual histories.
  python tools/diag_c3d.py perm strategy"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200 import gpc as G  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402

n = 24000
perm_no = int(sys.argv[1]) if len(sys.argv) > 1 else 4
strategy = sys.argv[2] if len(sys.argv) > 2 else "sym"
x, y = gpc_inputs(n, 8)
if perm_no:
    rng = np.random.default_rng(12345)
    perm = [rng.permutation(n) for _ in range(perm_no)][-1]
    x, y = x[perm], y[perm]
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 2.0)).with_strategy(strategy)
cfg = P.SolverConfig(tol=1e-8, ell=36)
st0 = G._make_state_dev(gram, torch.from_numpy(y).cuda())
# the pipelined loop of gpc._laplace_newton_pipelined without the NoProgress check
seq = P.SequenceState(k=32, cfg=cfg, selection="largest")
state = st0
system = G.build_newton_system(state)
for it in range(1, 4):
    x, job = P.recycle.solve_next_async(seq, system.a_matrix, system.b, ax0=system.ax0, ax0_of=system.x_prev)
    new_state, objective = G._update_dev_async(state, system.inner, system.sqrt_h, x)
    next_system = G.build_newton_system(new_state, x_prev=x) if it < 3 else None
    x, seq = job.finish()
    rep = seq.history[-1]
    _, psi = objective.get()
    A = system.a_matrix.with_strategy("rows")
    true = float(torch.linalg.norm(system.b - A.matvec_dev(x)) / torch.linalg.norm(system.b))
    h = rep.residual_history
    kb = None if seq.basis is None else seq.basis.k
    print(strategy, perm_no, os.environ.get("DCG_LIB_PATH"), "its", rep.iterations, "psi", psi, "rel", h[-1],
          "true", true, "next k", kb, "hist", [f"{v:.2e}" for v in h[:6]], "...", [f"{v:.2e}" for v in h[-3:]],
          flush=True)
    state, system = new_state, next_system
