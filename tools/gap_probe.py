"""Find the largest device-idle gap of a single-GPU config-3 Newton sequence and list the
host-side runtime calls (torch.profiler CPU + CUDA-runtime records) that overlap it.
  python tools/gap_probe.py [n] [reps]"""
import os, sys
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
d, ell, k = (8, 2.0, 32) if n >= 20000 else (10, 1.5, 16)
x, y = gpc_inputs(n, d, 0)
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, ell))
yd = torch.from_numpy(y).cuda()
cfg = P.SolverConfig(tol=1e-8, ell=k + 4)
run = lambda: P.laplace_newton(gram, yd, "defcg", cfg, newton_tol=-np.inf, max_newton=8, k=k, selection="largest")
run()
torch.cuda.synchronize()
for rep in range(reps):
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        recs = run()[1]
        torch.cuda.synchronize()
    dev = sorted(((e.time_range.start, e.time_range.end, e.name) for e in prof.events() if e.device_type.name == "CUDA"))
    cpu = sorted(((e.time_range.start, e.time_range.end, e.name) for e in prof.events() if e.device_type.name == "CPU"))
    t0 = dev[1][0]
    cur, gaps = dev[1][1], []
    for s, e, nme in dev[2:]:
        if s > cur:
            gaps.append((s - cur, cur, s, nme))
        cur = max(cur, e)
    gaps.sort(reverse=True)
    print("  solves ms:", [round((e - s) / 1e3, 2) for s, e, nme in dev if "dcg_solve_kernel" in nme], "iterations", [r.solver_iterations for r in recs])
    solve_ms = sum(e - s for s, e, nme in dev if "dcg_solve_kernel" in nme) / 1e3
    print(f"rep {rep}: solve kernels {solve_ms:.1f} ms; span {(cur - t0) / 1e3:.1f} ms; largest gaps:", [(round(g[0]), round((g[1] - t0) / 1e3, 1)) for g in gaps[:4]])
    g, a, b, nme = gaps[0]
    if g > 2000:
        print(f"  gap of {g:.0f} us from {(a - t0) / 1e3:.2f} ms, before {nme[:60]}; host records overlapping it (>= 50 us):")
        for s, e, cn in cpu:
            if e > a - 500 and s < b + 500 and e - s >= 50:
                print(f"    {(s - t0) / 1e3:10.2f} ms  {e - s:10.0f} us  {cn[:90]}")
