"""Host timing of the pieces before the first solve of laplace_newton, after a
gc.collect() (the bench's e2e first-step outliers)."""
import gc, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200 import gpc as G  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
x, y = gpc_inputs(10_000, 10)
xh, yh = torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory()
cfg = P.SolverConfig(tol=1e-8, ell=20)
T = {}
orig = {k: getattr(G, k) for k in ("_make_state_dev", "build_newton_system", "_pipelined_loop")}
def wrap(name):
    f = orig[name]
    def g(*a, **kw):
        t = time.perf_counter(); out = f(*a, **kw); T.setdefault(name, []).append((time.perf_counter() - t) * 1e3); return out
    setattr(G, name, g)
for k in orig: wrap(k)
for i in range(8):
    if i in (3, 6):
        gc.collect()
    torch.cuda.synchronize(); T.clear()
    t = time.perf_counter()
    xg, yg = xh.to("cuda", non_blocking=True), yh.to("cuda", non_blocking=True)
    t1 = time.perf_counter()
    g2 = P.rbf_kernel(xg, P.KernelParams(1.0, 1.5))
    t2 = time.perf_counter()
    st, recs = P.laplace_newton(g2, yg, "defcg", cfg, newton_tol=-np.inf, max_newton=8, k=16, selection="largest")
    t3 = time.perf_counter()
    st.f.cpu(); torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"iter {i}{' (after gc.collect)' if i in (3, 6) else ''}: h2d {1e3*(t1-t):.2f} rbf {1e3*(t2-t1):.2f} newton {1e3*(t3-t2):.2f} tail {1e3*(t4-t3):.2f} ms; "
          + " ".join(f"{k}={v[0]:.2f}" for k, v in T.items()))
