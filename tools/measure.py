#!/usr/bin/env python
"""Secondary measurements of the def-CG hot path (not the driver's bench line).

  python tools/measure.py config1        GPC Newton sequence n=2000, k=8 (BASELINE configs[0])
  python tools/measure.py config2-cg     config 2 with plain CG (k=0) for the def-CG vs CG comparison
  python tools/measure.py config4 [n]    GP-regression hyperparameter sweep, 20 lengthscales, k=24
  python tools/measure.py config3 [n]    GPC Newton sequence n=50000, d=8, ell=2, k=32, stored Gram (20 GB), 1 GPU
  python tools/measure.py config5 [n]    matrix-free RBF operator (K7), d=16, ell=3, k=32 (1 GPU)

Each prints one JSON line: device time (CUDA events) of the whole sequence,
iterations, iterations/s, and a CPU sample of the reference algorithm (oracle
port, numpy backend, all host threads) on the same inputs.  Inputs are the
seeded synthetic recipes of SURVEY.md section 8d.
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def gpc_sequence(n, d, ell, k, solver="defcg", reps=3, ell_log=None):
    import torch

    import paper_1706_00241_b200 as P
    from paper_1706_00241_b200.workloads import gpc_inputs

    x, y = gpc_inputs(n, d, 0)
    gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, ell))
    yd = torch.from_numpy(y).cuda()
    cfg = P.SolverConfig(tol=1e-8, ell=ell_log if ell_log is not None else max(k, 8) + 4)

    def run():
        _, recs = P.laplace_newton(gram, yd, solver, cfg, newton_tol=-np.inf, max_newton=8, k=k,
                                   selection="largest")
        return recs

    run()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        recs = run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    its = [r.solver_iterations for r in recs]
    return {"n": n, "k": k, "solver": solver, "iterations": its, "sequence_ms": best,
            "iters_per_s": sum(its) / (best / 1e3), "psi": [r.psi for r in recs]}


def cpu_gpc(n, d, ell, k, steps):
    from oracle import defcg_oracle as O

    x, y = O.gpc_inputs(n, d, 0)
    kmat = O.rbf_kernel(x, 1.0, ell, be="numpy")
    _, _, recs = O.laplace_newton(kmat, y, "defcg", O.Cfg(tol=1e-8, ell=k + 4), newton_tol=-np.inf, max_newton=8,
                                  k=k, selection="largest", be="numpy", max_steps_timed=steps)
    its = sum(r.solver_iterations for r in recs)
    secs = sum(r.solve_time_s for r in recs)
    return {"value": its / secs, "unit": "iters/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"first {len(recs)} Newton systems, {its} iterations in {secs:.2f} s"}


def sweep(n, k=24, n_theta=20, reps=1):
    import torch

    import paper_1706_00241_b200 as P
    from oracle.defcg_oracle import sweep_inputs

    x, y = sweep_inputs(n, d=8, seed=0)
    thetas = np.logspace(np.log10(0.5), np.log10(2.0), n_theta)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    cfg = P.SolverConfig(tol=1e-8, ell=k + 4)
    P.hyperparameter_sweep(xd, yd, thetas[:2], k=k, cfg=cfg)   # warm-up (allocations, contexts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, recs = P.hyperparameter_sweep(xd, yd, thetas, k=k, cfg=cfg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    e0.record()
    _, recs0 = P.hyperparameter_sweep(xd, yd, thetas, k=0, cfg=cfg)
    e1.record()
    torch.cuda.synchronize()
    ms0 = e0.elapsed_time(e1)
    its, its0 = [r.iterations for r in recs], [r.iterations for r in recs0]
    return {"n": n, "k": k, "thetas": len(thetas), "iterations": its, "sweep_ms": ms,
            "iters_per_s": sum(its) / (ms / 1e3), "plain_cg_iterations": its0, "plain_cg_sweep_ms": ms0,
            "includes": "Gram assembly per theta (K6) + refresh + def-CG + extraction"}


def cpu_sweep_sample(n, iters=5, n_cpu=12000):
    """Per-iteration CPU cost of the reference algorithm (numpy matvec on the
    host Gram, all threads), timed on `iters` CG iterations at n_cpu <= n and
    extrapolated proportionally to n^2 (the numpy Gram assembly needs several
    n x n temporaries, ~40 GB of host RAM at n = 30000)."""
    from oracle import defcg_oracle as O

    m = min(n, n_cpu)
    x, y = O.sweep_inputs(m, d=8, seed=0)
    a = O.rbf_kernel(x, 1.0, 0.5, jitter=0.01, be="numpy")
    t0 = time.perf_counter()
    _, rep, _ = O.cg_solve(a, y, None, O.Cfg(tol=1e-30, max_iters=iters, ell=0), be="numpy")
    dt = time.perf_counter() - t0
    scale = (m / n) ** 2
    return {"value": rep.iterations / dt * scale, "unit": "iters/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"{rep.iterations} plain-CG iterations at n={m} (numpy, all threads)"
                      + (f", extrapolated x(n_cpu/n)^2 = {scale:.3f} to n={n}" if m < n else "")}


def config5(n, d=16, ell=3.0, k=32, iters=20):
    """Matrix-free RBF operator (K7) at n points: device time of one product
    (CUDA events), FLOP_alg per product n^2 (2d + 4) (exp
    counted separately), and a def-CG solve of the first GPC Newton system
    with a random k-column basis (iterations, time per iteration)."""
    import torch

    import paper_1706_00241_b200 as P
    from paper_1706_00241_b200.workloads import gpc_inputs

    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal((n, d))).cuda()
    op = P.rbf_kernel(x, P.KernelParams(1.0, ell), matrix_free=True)
    v = torch.from_numpy(rng.standard_normal(n)).cuda()
    y = op.matvec_dev(v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        op.matvec_dev(v, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    # SURVEY 8d contract model: (2d + 4) flop per UNIQUE pair, n (n + 1) / 2 pairs
    flop = float(n) * (n + 1) / 2 * (2 * d + 4)
    s = torch.from_numpy(rng.uniform(0.2, 0.5, n)).cuda()
    a = op.scaled(s, 1.0)
    b = torch.from_numpy(rng.standard_normal(n)).cuda()
    cfg = P.SolverConfig(tol=1e-8, ell=k + 4, max_iters=iters)
    wk = torch.from_numpy(rng.standard_normal((n, k))).cuda()
    basis = P.refresh_basis(a, wk)
    torch.cuda.synchronize()
    e0.record()
    basis = P.refresh_basis(a, wk)
    e1.record()
    torch.cuda.synchronize()
    refresh_ms = e0.elapsed_time(e1)
    half = a.with_rows(0, n // 2) if hasattr(a, "with_rows") else None
    del half
    _, rep, _ = P.deflated_cg_solve(a, b, torch.zeros(n, dtype=torch.float64, device="cuda"), basis, cfg)
    dmma_peak = 37.1   # TFLOP/s, tools/fp64_peak.cu on this B200 (FP64 tensor pipe)
    return {"n": n, "d": d, "matvec_ms": ms, "flop_alg_per_matvec": flop, "achieved_tflops": flop / (ms / 1e3) / 1e12,
            "frac_of_fp64_peak": flop / (ms / 1e3) / 1e12 / dmma_peak, "flop_model": "(2d+4) n(n+1)/2 (SURVEY 8d)",
            "exp_per_s": float(n) * (n + 1) / 2 / (ms / 1e3), "solve_iterations": rep.iterations,
            "solve_ms_per_iteration": rep.device_ms / (rep.iterations + 2),
            "refresh_ms_k": [refresh_ms, k],
            "note": "symmetric half-evaluation (each pair once), dot-product distance form"}


def config5_slab(n=200000, d=16, ell=3.0, k=32, world=8):
    """Config 5 per rank: rank 0's row slab (n / world rows) of the matrix-free
    operator -- the product every rank runs per sharded def-CG iteration, and
    the slab's multi-vector product of the refresh (k columns)."""
    import ctypes

    import torch

    import paper_1706_00241_b200 as P
    from paper_1706_00241_b200.sharded import sharded_rbf_kernel

    C = type("C", (), {"rank": 0, "world": world})

    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal((n, d))).cuda()
    s = torch.from_numpy(rng.uniform(0.2, 0.5, n)).cuda()
    op = sharded_rbf_kernel(x, P.KernelParams(1.0, ell), comm=C(), matrix_free=True).scaled(s, 1.0)
    c = op.c_struct()
    v = torch.from_numpy(rng.standard_normal(n)).cuda()
    w = torch.from_numpy(rng.standard_normal((n, k))).cuda()
    y = torch.empty(op.rows, dtype=torch.float64, device="cuda")
    yb = torch.empty(op.rows, k, dtype=torch.float64, device="cuda")
    lib, ctx, st = P._native.lib(), P._device.ctx(), P._device.stream()

    def apply():
        P._native.check(lib.dcg_op_apply(ctx, st, ctypes.byref(c), v.data_ptr(), y.data_ptr()))

    def block():
        P._native.check(lib.dcg_op_apply_block(ctx, st, ctypes.byref(c), w.data_ptr(), k, yb.data_ptr()))

    t = torch.empty(n, dtype=torch.float64, device="cuda")

    def sym_share(rank):
        def fn():
            P._native.check(lib.dcg_shard_rbf_sym_partial(ctx, st, ctypes.byref(c), rank, world, v.data_ptr(),
                                                          t.data_ptr(), None))
        return fn

    out = {"n": n, "d": d, "k": k, "world": world, "rows_per_rank": op.rows}
    for name, fn, reps in (("slab_matvec_ms", apply, 3), ("slab_block_ms", block, 1),
                           ("sym_share_rank0_ms", sym_share(0), 3), (f"sym_share_rank{world - 1}_ms",
                                                                      sym_share(world - 1), 3)):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / reps
    pairs = float(n) * op.rows
    ops = pairs * (d + 12 + 1)
    out["slab_fp64_ops_per_s"] = ops / (out["slab_matvec_ms"] / 1e3)
    out["sym_allreduce_bytes"] = 8 * n
    out["note"] = ("sym_share: this rank's share of the lower-triangle tiles (each pair once) + local pass 2, "
                   "followed by an all-reduce of 8n bytes; slab_*: "
                   "row-owned tensor-pipe kernel (rbf_mma_rows_kernel): per element d DMMA-FMAs + ~12 FP64 ops "
                   "(exp, init) + 1 (product) [+ k on DMMA for the block product]; each rank also all-gathers p "
                   "(8n B) per iteration")
    return out


def config5_sequence(n=200000, steps=8, d=16, ell=3.0, k=32, ell_log=36):
    """BASELINE config 5 at one GPU: the GPC Newton sequence on the matrix-free
    RBF operator (K regenerated tile by tile in every product; the 320 GB
    Gram is never stored), def-CG with k = 32, one timed sequence (CUDA
    events) after the operand set-up."""
    import torch

    import paper_1706_00241_b200 as P
    from paper_1706_00241_b200.workloads import gpc_inputs

    x, y = gpc_inputs(n, d, 0)
    op = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, ell), matrix_free=True)
    yd = torch.from_numpy(y).cuda()
    cfg = P.SolverConfig(tol=1e-8, ell=ell_log)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    _, recs = P.laplace_newton(op, yd, "defcg", cfg, newton_tol=-np.inf, max_newton=steps, k=k, selection="largest")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    its = [r.solver_iterations for r in recs]
    pairs = n * (n + 1) / 2
    return {"n": n, "d": d, "lengthscale": ell, "k": k, "ell_log": ell_log, "newton_steps": steps,
            "iterations": its, "sequence_ms": ms, "iters_per_s": sum(its) / (ms / 1e3),
            "psi": [r.psi for r in recs], "wall_s": time.perf_counter() - t0,
            "pairs_per_product": pairs, "note": "matrix-free (Gram never stored), one GPU, CUDA events"}


def main():
    what = sys.argv[1]
    if what == "config1":
        out = gpc_sequence(2000, 5, 1.5, 8)
        out["cpu_baseline"] = cpu_gpc(2000, 5, 1.5, 8, 8)
    elif what == "config2-cg":
        out = {"defcg": gpc_sequence(10000, 10, 1.5, 16), "cg": gpc_sequence(10000, 10, 1.5, 0, solver="cg")}
    elif what == "config4":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 30000
        out = sweep(n)
        out["cpu_baseline"] = cpu_sweep_sample(n)
    elif what == "config3":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
        out = gpc_sequence(n, 8, 2.0, 32, reps=1, ell_log=36)
        out["gram_bytes"] = 8 * n * n
        out["note"] = "BASELINE configs[2] at one GPU (the 1-GPU point of its 1/2/4/8 scaling); stored Gram in HBM"
        out["cpu_baseline"] = cpu_sweep_sample(n, n_cpu=12000)
        out["cpu_baseline"]["sample"] += " (plain-CG iteration cost on the host at n_cpu, scaled to n)"
    elif what == "config5-slab":
        out = config5_slab(int(sys.argv[2]) if len(sys.argv) > 2 else 200000)
    elif what == "config5":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
        out = config5(n)
    elif what == "config5-seq":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 200000
        steps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
        out = config5_sequence(n, steps)
    else:
        raise SystemExit(__doc__)
    out["workload"] = what
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
