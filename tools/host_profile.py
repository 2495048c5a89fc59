"""Host-side time per section of the pipelined config-2 Newton loop (what the
GPU waits on when the host is late): wraps the pieces of
gpc._laplace_newton_pipelined with perf_counter stamps."""
import collections, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200 import gpc as G, recycle as R  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402

acc = collections.defaultdict(list)


def wrap(mod, name, label):
    f = getattr(mod, name)

    def g(*a, **kw):
        t = time.perf_counter()
        out = f(*a, **kw)
        acc[label].append((time.perf_counter() - t) * 1e6)
        return out
    setattr(mod, name, g)


wrap(G, "solve_next_async", "solve_next_async")
wrap(G, "_update_dev_async", "update_dev_async")
wrap(G, "build_newton_system", "build_newton_system")
fin = R._AsyncSolve.finish


def fin_w(self, *a, **kw):
    t = time.perf_counter()
    out = fin(self, *a, **kw)
    acc["job.finish"].append((time.perf_counter() - t) * 1e6)
    return out


R._AsyncSolve.finish = fin_w
og = G._PendingObjective.get


def og_w(self):
    t = time.perf_counter()
    out = og(self)
    acc["objective.get"].append((time.perf_counter() - t) * 1e6)
    return out


G._PendingObjective.get = og_w
x, y = gpc_inputs(10_000, 10)
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.5))
yd = torch.from_numpy(y).cuda()
cfg = P.SolverConfig(tol=1e-8, ell=20)
for _ in range(3):
    P.laplace_newton(gram, yd, "defcg", cfg, newton_tol=-np.inf, max_newton=8, k=16, selection="largest")
acc.clear()
torch.cuda.synchronize()
t = time.perf_counter()
P.laplace_newton(gram, yd, "defcg", cfg, newton_tol=-np.inf, max_newton=8, k=16, selection="largest")
torch.cuda.synchronize()
print(f"sequence wall {1e3 * (time.perf_counter() - t):.2f} ms")
for k, v in acc.items():
    print(f"{k:22s} n={len(v)} mean {np.mean(v):8.1f} us  per call {[round(u) for u in v]}")
