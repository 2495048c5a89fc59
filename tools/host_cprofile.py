"""cProfile of the host side of the pipelined config-2 Newton loop."""
import cProfile, os, pstats, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
x, y = gpc_inputs(10_000, 10)
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.5))
yd = torch.from_numpy(y).cuda()
cfg = P.SolverConfig(tol=1e-8, ell=20)
run = lambda: P.laplace_newton(gram, yd, "defcg", cfg, newton_tol=-np.inf, max_newton=8, k=16, selection="largest")
for _ in range(3):
    run()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    run()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumulative").print_stats(40)
