"""Host time of the head of a config-2 Newton sequence (before the first solve
kernel can start): state init, first system, first solve enqueue."""
import os, sys, time, statistics as S
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200 import gpc as G  # noqa: E402
from paper_1706_00241_b200.recycle import solve_next_async  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
x, y = gpc_inputs(10_000, 10)
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.5))
yd = torch.from_numpy(y).cuda()
cfg = P.SolverConfig(tol=1e-8, ell=20)
run = lambda: P.laplace_newton(gram, yd, "defcg", cfg, newton_tol=-np.inf, max_newton=8, k=16, selection="largest")
for _ in range(3):
    run()
torch.cuda.synchronize()
rows = []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    state = G._make_state_dev(gram, yd)
    t1 = time.perf_counter()
    seq = P.SequenceState(k=16, cfg=cfg, selection="largest")
    system = G.build_newton_system(state)
    t2 = time.perf_counter()
    xs, job = solve_next_async(seq, system.a_matrix, system.b, extract=True, need_aw=False)
    t3 = time.perf_counter()
    new_state, objective = G._update_dev_async(state, system.inner, system.sqrt_h, xs)
    t4 = time.perf_counter()
    nxt = G.build_newton_system(new_state, x_prev=xs)
    t5 = time.perf_counter()
    from paper_1706_00241_b200.recycle import prepare_refresh
    prep = prepare_refresh(job, nxt.a_matrix)
    t6 = time.perf_counter()
    job.finish()
    torch.cuda.synchronize()
    rows.append([(b - a) * 1e6 for a, b in ((t0, t1), (t1, t2), (t2, t3), (t3, t4), (t4, t5), (t5, t6))])
names = ["make_state(sync)", "build_system", "solve_next_async", "update_async", "next_system", "prepare_refresh"]
for i, nme in enumerate(names):
    print(f"{nme:20s} median {S.median(r[i] for r in rows):8.1f} us  min {min(r[i] for r in rows):8.1f}")
# whole sequences, wall vs device
ts = []
for _ in range(10):
    torch.cuda.synchronize(); t0 = time.perf_counter(); run(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
print("sequence wall ms:", " ".join(f"{t:.2f}" for t in ts))
