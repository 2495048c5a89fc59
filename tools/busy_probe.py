"""Device-busy share and the largest idle gaps (torch.profiler / CUPTI) of a workload:
  python tools/busy_probe.py sweep [n] [thetas] | mf [n] [steps] | config1
Prints per-kernel totals, the busy share of the span, memcpy totals and the largest gaps."""
import collections, os, sys
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
what = sys.argv[1] if len(sys.argv) > 1 else "sweep"
if what == "sweep":
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30000
    nt = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal((n, 8))).cuda()
    y = torch.from_numpy(rng.standard_normal(n)).cuda()
    thetas = P.default_lengthscales()[:nt]
    cfg = P.SolverConfig(tol=1e-8, ell=28)
    run = lambda: P.hyperparameter_sweep(x, y, thetas, k=24, cfg=cfg)
elif what == "mf":
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    xx, yy = gpc_inputs(n, 16, 0)
    op = P.rbf_kernel(torch.from_numpy(xx).cuda(), P.KernelParams(1.0, 3.0), matrix_free=True)
    yd = torch.from_numpy(yy).cuda()
    cfg = P.SolverConfig(tol=1e-8, ell=36)
    run = lambda: P.laplace_newton(op, yd, "defcg", cfg, newton_tol=-np.inf, max_newton=steps, k=32, selection="largest")
else:
    xx, yy = gpc_inputs(2000, 5, 0)
    gram = P.rbf_kernel(torch.from_numpy(xx).cuda(), P.KernelParams(1.0, 1.0))
    yd = torch.from_numpy(yy).cuda()
    cfg = P.SolverConfig(tol=1e-8, ell=12)
    run = lambda: P.laplace_newton(gram, yd, "defcg", cfg, newton_tol=-np.inf, max_newton=8, k=8, selection="largest")
run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
evs = sorted(((e.time_range.start, e.time_range.end, e.name) for e in prof.events() if e.device_type.name == "CUDA"))
evs = evs[1:] if len(evs) > 2 and evs[1][0] - evs[0][1] > 500 else evs   # (a stale first record)
t0, t1 = evs[0][0], max(e[1] for e in evs)
tot = collections.defaultdict(lambda: [0.0, 0])
for s, e, nme in evs:
    tot[nme[:64]][0] += e - s
    tot[nme[:64]][1] += 1
print(f"{what}: span {(t1 - t0) / 1e3:.2f} ms, {len(evs)} device events")
for k, (v, c) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:16]:
    print(f"{v / 1e3:10.3f} ms {c:6d}  {k}")
busy, cur, gaps = 0.0, t0, []
for s, e, nme in evs:
    if s > cur:
        gaps.append((s - cur, cur - t0, nme[:50]))
        busy += e - s
        cur = e
    elif e > cur:
        busy += e - cur
        cur = e
print(f"device busy {busy / 1e3:.2f} ms = {100 * busy / (t1 - t0):.1f}% of span")
for g, at, nme in sorted(gaps, key=lambda t: -t[0])[:10]:
    print(f"  gap {g:9.1f} us at {at / 1e3:9.2f} ms before {nme}")
