"""Per-phase device time of dcg_shard_step (DCG_STEP_TIMERS, CTA 0) over one sharded config-3 sequence at world 1."""
import ctypes, os, sys
os.environ["DCG_STEP_TIMERS"] = "1"
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200 import _native as N  # noqa: E402
from paper_1706_00241_b200.sharded import SelfComm, sharded_laplace_newton, sharded_rbf_kernel  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
x, y = gpc_inputs(n, 8)
op = sharded_rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 2.0), None, SelfComm())
recs = sharded_laplace_newton(op, torch.from_numpy(y).cuda(), None, P.SolverConfig(tol=1e-8, ell=36), newton_tol=-np.inf,
                              max_newton=4, k=32, selection="largest", comm=SelfComm())
torch.cuda.synchronize()
its = sum(r.solver_iterations for r in recs)
out = (ctypes.c_ulonglong * 16)()
lib = ctypes.CDLL(str(N.LIB_PATH))
assert lib.dcg_debug_step_timers(out) == 0
names = ["epilogue+pAp", "barrier1", "d sum", "x,r", "row partials", "barrier2", "reduce", "mu", "p"]
print("iterations", its, " us per step:", "  ".join(f"{nm}={out[i] / 1e3 / its:.2f}" for i, nm in enumerate(names)),
      f" total={sum(out[:9]) / 1e3 / its:.2f}")
