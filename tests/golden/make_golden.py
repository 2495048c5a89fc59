"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory, builds the reference's
Cython kernel core there (``setup.py build_ext --inplace``; no reference
source is copied into this repo), imports ``defcg`` from that copy and records
its outputs on seeded inputs into ``tests/golden/*.npz``.  Both kernel
backends are recorded where they differ ("compiled" is the reference default,
"numpy" its fallback) so tests can state the reference's own noise floor.
These fixtures travel with the repo; nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import importlib
import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg")


def load_reference(backend: str):
    scratch = Path(tempfile.gettempdir()) / "defcg_ref_golden"
    if not (scratch / "src" / "defcg" / "_kernels").exists() or not list((scratch / "src" / "defcg" / "_kernels").glob("_core*.so")):
        if scratch.exists():
            shutil.rmtree(scratch)
        shutil.copytree(REF, scratch)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=scratch, check=True,
                       capture_output=True)
    os.environ["DEFCG_BACKEND"] = backend
    for name in list(sys.modules):
        if name == "defcg" or name.startswith("defcg."):
            del sys.modules[name]
    sys.path.insert(0, str(scratch / "src"))
    try:
        mod = importlib.import_module("defcg")
    finally:
        sys.path.pop(0)
    assert mod.BACKEND == backend, (mod.BACKEND, backend)
    return mod


def random_spd(rng, n, kappa=100.0):
    """Same construction as the reference test suite's conftest (log-spaced spectrum)."""
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    a = q @ np.diag(np.logspace(0.0, np.log10(kappa), n)) @ q.T
    return 0.5 * (a + a.T)


def gpc_inputs(n, d, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d))
    noise = rng.standard_normal(n)
    t = np.sin(2.0 * x).sum(axis=1) + 0.1 * noise
    return x, np.where(t >= 0.0, 1.0, -1.0)


def kernels(dc, tag):
    from defcg import _kernels as K

    rng = np.random.default_rng(11)
    out = {}
    a = rng.standard_normal((37, 29))
    x = rng.standard_normal(29)
    b = rng.standard_normal((29, 7))
    out["mv_a"], out["mv_x"], out["mv_y"] = a, x, K.matvec(a, x)
    out["gemm_b"], out["gemm_c"] = b, K.gemm(a, b)
    s = random_spd(rng, 23, 1e3)
    low, fail = K.cholesky(s, 1e-14 * np.max(np.diag(s)))
    out["chol_a"], out["chol_l"], out["chol_fail"] = s, low, np.array(fail)
    ind = np.array([[1.0, 2.0], [2.0, 1.0]])
    _, fail2 = K.cholesky(ind, 1e-14)
    out["chol_ind_fail"] = np.array(fail2)
    rhs = rng.standard_normal(23)
    out["sl_b"], out["sl_y"], out["slt_x"] = rhs, K.solve_lower(low, rhs), K.solve_lower_trans(low, rhs)
    pts = rng.standard_normal((41, 6))
    out["rbf_x"], out["rbf_k"] = pts, K.rbf_gram(pts, 1.7, 1.0 / (2 * 1.3**2), 1e-3)
    jac = random_spd(rng, 17, 50.0)
    jv = np.eye(17)
    work = jac.copy()
    out["jac_a"] = jac
    out["jac_rot"] = np.array(K.jacobi_sweep(work, jv))
    out["jac_a1"], out["jac_v1"] = work, jv
    return {f"{tag}_{k}": v for k, v in out.items()}


def solvers(dc, tag):
    from defcg.recycle import refresh_basis
    from defcg.solvers import SolverConfig, cg_solve, deflated_cg_solve

    rng = np.random.default_rng(21)
    out = {}
    for case, (n, kappa, k, tol, ell) in enumerate([(30, 1e3, 0, 1e-10, 8), (40, 1e4, 3, 1e-10, 12),
                                                    (25, 1e2, 5, 1e-12, 30), (60, 1e5, 4, 1e-8, 6)]):
        a = random_spd(rng, n, kappa)
        bvec = rng.standard_normal(n)
        x_prev = rng.standard_normal(n)
        cfg = SolverConfig(tol=tol, ell=ell)
        p = f"c{case}_"
        out[p + "a"], out[p + "b"], out[p + "xprev"] = a, bvec, x_prev
        out[p + "cfg"] = np.array([tol, ell, k])
        if k == 0:
            x, rep, log = cg_solve(a, bvec, x_prev, cfg)
        else:
            w = rng.standard_normal((n, k))
            basis = refresh_basis(a, w)
            out[p + "w"] = w
            out[p + "chol"] = basis.gram_chol
            out[p + "aw"] = basis.aw
            x, rep, log = deflated_cg_solve(a, bvec, x_prev, basis, cfg)
        out[p + "x"] = x
        out[p + "hist"] = np.array(rep.residual_history)
        out[p + "its"] = np.array(rep.iterations)
        out[p + "logp"] = np.array(log.p)
        out[p + "logr"] = np.array(log.r)
        out[p + "alpha"] = np.array(log.alpha)
        out[p + "beta"] = np.array(log.beta)
        out[p + "d"] = np.array(log.d)
        if k:
            out[p + "mu"] = np.array(log.mu)
    # a 60-iteration solve crossing the true-residual refresh (every 50)
    a = random_spd(rng, 120, 1e6)
    bvec = rng.standard_normal(120)
    x, rep, _ = cg_solve(a, bvec, None, SolverConfig(tol=1e-12, ell=4))
    out["long_a"], out["long_b"], out["long_x"] = a, bvec, x
    out["long_hist"] = np.array(rep.residual_history)
    return {f"{tag}_{k}": v for k, v in out.items()}


def recycle(dc, tag):
    from defcg.recycle import SequenceState, harmonic_ritz_extract, refresh_basis, solve_next
    from defcg.solvers import SolverConfig, cg_solve

    rng = np.random.default_rng(31)
    out = {}
    a = random_spd(rng, 50, 1e4)
    bvec = rng.standard_normal(50)
    _, rep, log = cg_solve(a, bvec, None, SolverConfig(tol=1e-10, ell=12))
    for sel in ("smallest", "largest"):
        ext = harmonic_ritz_extract(log, None, 5, sel)
        out[f"ritz_{sel}_theta"] = ext.theta
        out[f"ritz_{sel}_w"] = ext.w_next
        out[f"ritz_{sel}_aw"] = ext.aw_next
    out["ritz_a"], out["ritz_b"] = a, bvec
    # refresh with a dependent column -> pruned to k-1
    w = rng.standard_normal((50, 3))
    w = np.hstack([w, w[:, [1]]])
    basis = refresh_basis(a, w)
    out["refresh_w_in"], out["refresh_w"], out["refresh_aw"], out["refresh_chol"] = w, basis.w, basis.aw, basis.gram_chol
    # a short sequence of perturbed systems
    st = SequenceState(k=4, cfg=SolverConfig(tol=1e-9, ell=10), selection="largest")
    mats, rhs, xs, its = [], [], [], []
    base = random_spd(rng, 64, 1e4)
    for step in range(4):
        jit = 0.01 * random_spd(rng, 64, 2.0)
        am = 0.5 * (base + base.T) + jit
        bb = rng.standard_normal(64)
        x, st = solve_next(st, am, bb)
        mats.append(am)
        rhs.append(bb)
        xs.append(x)
        its.append(st.history[-1].iterations)
    out["seq_a"], out["seq_b"], out["seq_x"], out["seq_its"] = np.array(mats), np.array(rhs), np.array(xs), np.array(its)
    return {f"{tag}_{k}": v for k, v in out.items()}


def gpc(dc, tag, n=2000, d=5, ell=1.5, k=8):
    from defcg.gpc import KernelParams, laplace_newton, rbf_kernel
    from defcg.solvers import SolverConfig

    x, y = gpc_inputs(n, d)
    kmat = rbf_kernel(x, KernelParams(1.0, ell))
    out = {"x": x, "y": y}
    for solver in ("cg", "defcg"):
        _, recs = laplace_newton(kmat, y, solver, SolverConfig(tol=1e-8, ell=k + 4), newton_tol=-np.inf,
                                 max_newton=8, k=k, selection="largest")
        out[f"{solver}_its"] = np.array([r.solver_iterations for r in recs])
        out[f"{solver}_psi"] = np.array([r.psi for r in recs])
        out[f"{solver}_rel"] = np.array([r.rel_residual for r in recs])
        out[f"{solver}_f"] = recs[-1].f
        out[f"{solver}_f1"] = recs[0].f
    return {f"{tag}_{k2}": v for k2, v in out.items()}


def main():
    meta = {"numpy": np.__version__}
    for backend in ("compiled", "numpy"):
        dc = load_reference(backend)
        tag = "c" if backend == "compiled" else "n"
        np.savez_compressed(OUT / f"kernels_{backend}.npz", **kernels(dc, tag))
        np.savez_compressed(OUT / f"solvers_{backend}.npz", **solvers(dc, tag))
        np.savez_compressed(OUT / f"recycle_{backend}.npz", **recycle(dc, tag))
        np.savez_compressed(OUT / f"gpc_small_{backend}.npz", **gpc(dc, tag, n=300, d=4, ell=1.2, k=4))
        np.savez_compressed(OUT / f"config1_{backend}.npz", **gpc(dc, tag))
        if os.environ.get("GOLDEN_CONFIG2", "1") == "1":
            g2 = gpc(dc, tag, n=10_000, d=10, ell=1.5, k=16)
            g2.pop(f"{tag}_x")   # regenerated from the seed at test time
            np.savez_compressed(OUT / f"config2_{backend}.npz", **g2)
        print("wrote goldens for backend", backend, flush=True)
    (OUT / "VERSIONS.txt").write_text(
        "generated by tests/golden/make_golden.py from /root/reference/pkg (defcg 0.1.0)\n"
        f"numpy {meta['numpy']}\n"
    )


if __name__ == "__main__":
    main()
