"""Per-phase device timers (DCG_PHASE_TIMERS, CTA 0, printed by the library on
stderr) of the first two solves of the config-2 sequence run through the
synchronous solve_next (plain CG, then def-CG with k = 16)."""
import os, sys
os.environ["DCG_PHASE_TIMERS"] = "1"
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200 import gpc as G  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
x, y = gpc_inputs(10_000, 10)
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.5))
cfg = P.SolverConfig(tol=1e-8, ell=20)
st = G.make_state(gram, torch.from_numpy(y).cuda())
seq = P.SequenceState(k=16, cfg=cfg, selection="largest")
for step in range(3):
    sysm = G.build_newton_system(st)
    xs, seq = P.solve_next(seq, sysm.a_matrix, sysm.b)
    st, _ = G._update_dev(st, sysm.inner, sysm.sqrt_h, xs)
    print("step", step + 1, "iterations", seq.history[-1].iterations, flush=True)
