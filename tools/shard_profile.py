"""Sharded Newton sequence at world 1 (SelfComm) on the config-3 recipe, for
kernel launch lists (ncu) of the tile-share path.  python tools/shard_profile.py [n] [steps]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200.sharded import SelfComm, sharded_laplace_newton, sharded_rbf_kernel  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
x, y = gpc_inputs(n, 8)
params = P.KernelParams(1.0, 2.0)
op = sharded_rbf_kernel(torch.from_numpy(x).cuda(), params, None, SelfComm())
recs = sharded_laplace_newton(op, torch.from_numpy(y).cuda(), None, P.SolverConfig(tol=1e-8, ell=36),
                              newton_tol=-np.inf, max_newton=steps, k=32, selection="largest", comm=SelfComm())
print([r.solver_iterations for r in recs])
