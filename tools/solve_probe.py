"""Per-iteration time of the persistent solve kernel on a GPC Newton system.

  python tools/solve_probe.py [n] [d] [lengthscale] [reps]

Builds the first Newton system of the config recipe (seeded inputs), runs
plain CG at rtol 1e-8 `reps` times, and prints the kernel's device time per
iteration (CUDA events around the cooperative launch), the iteration count
and the algorithmic HBM rate (8 n(n+1)/2 B per product).  Environment knobs
of the library apply (DCG_L2_PIN_MB, DCG_PHASE_TIMERS)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ell = float(sys.argv[3]) if len(sys.argv) > 3 else 1.5
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
x, y = gpc_inputs(n, d)
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, ell))
st0 = P.gpc.make_state(gram, torch.from_numpy(y).cuda())
sys0 = P.gpc.build_newton_system(st0)
x0 = torch.zeros(n, dtype=torch.float64, device="cuda")
cfg = P.SolverConfig(tol=1e-8, ell=0)
best, its, xs = None, None, None
for _ in range(reps):
    xs, rep, _ = P.cg_solve(sys0.a_matrix, sys0.b, x0, cfg)
    ms = rep.device_ms
    best = ms if best is None else min(best, ms)
    its = rep.iterations
products = its + 1
gram_bytes = 8 * n * (n + 1) / 2
vec = 8 * n * 10 * its
out = {"n": n, "iterations": its, "kernel_ms": best, "us_per_iteration": best * 1e3 / its,
       "alg_GBps": (products * gram_bytes + vec) / (best / 1e3) / 1e9, "pin_mb": os.environ.get("DCG_L2_PIN_MB"),
       "x_checksum": float(xs.sum())}
peaks = os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")
if os.path.exists(peaks):
    out["frac"] = out["alg_GBps"] / json.load(open(peaks))["hbm_gbs"]
print(json.dumps(out))
