#!/usr/bin/env python
"""One config-2 Newton sequence between cudaProfilerStart/Stop, after warm-up,
for `ncu --profile-from-start off` launch lists (profiles/).

  python tools/profile_seq.py [n] [solver]     (defaults: 10000 defcg)

Without a profiler it prints the wall time of each phase of the sequence
(host-side view, synchronised), which shows where the non-kernel time goes.
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import paper_1706_00241_b200 as P
    from oracle.defcg_oracle import gpc_inputs

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    solver = sys.argv[2] if len(sys.argv) > 2 else "defcg"
    x, y = gpc_inputs(n, 10, 0)
    gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.5))
    yd = torch.from_numpy(y).cuda()
    cfg = P.SolverConfig(tol=1e-8, ell=20)

    def run():
        return P.laplace_newton(gram, yd, solver, cfg, newton_tol=-np.inf, max_newton=8, k=16, selection="largest")

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, recs = run()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    torch.cuda.cudart().cudaProfilerStart()
    run()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print(f"n={n} solver={solver} iterations={[r.solver_iterations for r in recs]} wall={wall * 1e3:.2f} ms "
          f"solve_time={[round(r.solve_time_s * 1e3, 2) for r in recs]}")


if __name__ == "__main__":
    main()
