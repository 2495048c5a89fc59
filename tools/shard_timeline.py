"""GPU timeline (torch.profiler / CUPTI) of one sharded config-3 Newton sequence at
world 1 (tile-share path): per-kernel totals, device-busy share, the largest idle gaps.
  python tools/shard_timeline.py [n] [steps]"""
import collections, os, sys
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200.sharded import SelfComm, sharded_laplace_newton, sharded_rbf_kernel  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
x, y = gpc_inputs(n, 8)
op = sharded_rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 2.0), None, SelfComm())
yd = torch.from_numpy(y).cuda()
run = lambda: sharded_laplace_newton(op, yd, None, P.SolverConfig(tol=1e-8, ell=36), newton_tol=-np.inf,
                                     max_newton=steps, k=32, selection="largest", comm=SelfComm())
run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    recs = run()
    torch.cuda.synchronize()
evs = sorted(((e.time_range.start, e.time_range.end, e.name) for e in prof.events() if e.device_type.name == "CUDA"),
             key=lambda t: t[0])
t0, t1 = evs[0][0], max(e[1] for e in evs)
tot = collections.defaultdict(lambda: [0.0, 0])
for s, e, nme in evs:
    tot[nme[:70]][0] += e - s
    tot[nme[:70]][1] += 1
print("iterations", [r.solver_iterations for r in recs])
print(f"span {(t1 - t0) / 1e3:.2f} ms, {len(evs)} device events")
for k, (v, c) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:28]:
    print(f"{v / 1e3:10.3f} ms {c:6d}  {k}")
# busy time (union of intervals) and the largest gaps
busy, cur_e, gaps = 0.0, t0, []
for s, e, nme in evs:
    if s > cur_e:
        gaps.append((s - cur_e, cur_e - t0, nme[:50]))
        busy += e - s
        cur_e = e
    elif e > cur_e:
        busy += e - cur_e
        cur_e = e
print(f"device busy {busy / 1e3:.2f} ms = {100 * busy / (t1 - t0):.1f}% of span; idle {(t1 - t0 - busy) / 1e3:.2f} ms in {len(gaps)} gaps")
for g, at, nme in sorted(gaps, key=lambda t: -t[0])[:25]:
    print(f"  gap {g:9.1f} us at {at / 1e3:9.2f} ms before {nme}")
small = sum(g for g, _, _ in gaps if g < 20)
print(f"  gaps < 20 us: {small / 1e3:.2f} ms total")
