"""Per-iteration wall time of the bench's end-to-end step (pinned X, y ->
device, rbf_kernel, laplace_newton, records to the host), with the Python
garbage collector's activity."""
import gc, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
x, y = gpc_inputs(10_000, 10)
xh, yh = torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory()
cfg = P.SolverConfig(tol=1e-8, ell=20)
gcs = []
gc.callbacks.append(lambda phase, info: gcs.append((phase, info.get("generation"), time.perf_counter())))


def once():
    xg, yg = xh.to("cuda", non_blocking=True), yh.to("cuda", non_blocking=True)
    g2 = P.rbf_kernel(xg, P.KernelParams(1.0, 1.5))
    st, recs = P.laplace_newton(g2, yg, "defcg", cfg, newton_tol=-np.inf, max_newton=8, k=16, selection="largest")
    st.f.cpu()


for i in range(12):
    torch.cuda.synchronize()
    n0 = len(gcs)
    t = time.perf_counter()
    once()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) * 1e3
    mem = torch.cuda.memory_allocated() / 1e6
    print(f"iter {i}: {dt:7.2f} ms  gc events {len(gcs) - n0}  allocated {mem:8.1f} MB  reserved {torch.cuda.memory_reserved() / 1e6:8.1f} MB")
