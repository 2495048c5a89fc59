"""Golden vectors at the larger BASELINE configs, produced by running the REFERENCE itself.

Run in the build container (where /root/reference exists; ~62 GB host RAM):

    python tests/golden/make_golden_big.py [config3|config4|config5|config2tight|all]

Same mechanics as ``make_golden.py`` (the reference package is copied to a
scratch directory and its Cython core built there; nothing of the reference is
copied into this repo).  What it records, per config recipe of SURVEY.md §8d:

* ``config3_ref.npz`` -- config 3's recipe (X ~ N(0, I_8), lengthscale 2.0,
  k = 32, ell_log = 36, tol 1e-8) at n = 24,000 (the largest size whose
  reference run fits this host: the reference's peak RSS is ~4 x 8 n^2), the
  first 3 Newton steps: iteration counts, psi, final relative residuals, the
  latent f after step 1; for the compiled backend, the numpy backend, and the
  numpy backend on symmetric row permutations of the same data (the
  reference's own rounding spread of the counts).
* ``config4_ref.npz`` -- config 4 (GP-regression sweep, X ~ U[-1,1]^8,
  n = 30,000, jitter 0.01, k = 24, ell_log = 28), the first 3 lengthscales of
  the 20-point log grid: iteration counts and solutions, numpy backend (the
  compiled backend's single-core matvec would need ~1 s per iteration here),
  plus permuted runs for the spread.
* ``config5_ref.npz`` -- config 5's recipe (X ~ N(0, I_16), lengthscale 3.0,
  k = 32, ell_log = 36) at n = 16,000, the first 3 Newton steps; the GPU side
  runs it through the MATRIX-FREE operator.
* ``config2_tight_ref.npz`` -- the first Newton system of config 2 (n = 10^4)
  solved by the reference's cg_solve at rtol 1e-12 (SURVEY §7 hard part 1(b):
  the 1e-9 solution bar is checked on systems re-solved tightly), plus the
  config-3-recipe first system at n = 24,000 at rtol 1e-12.

Inputs are regenerated from the seeds at test time; only outputs are stored.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
from make_golden import OUT, gpc_inputs, load_reference  # noqa: E402

N_PERM = 4


def sweep_inputs(n, d=8, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1.0, 1.0, (n, d))
    noise = rng.standard_normal(n)
    return x, np.sin(3.0 * x).sum(axis=1) + 0.05 * noise


def perms(n, count):
    rng = np.random.default_rng(12345)
    return [rng.permutation(n) for _ in range(count)]


def gpc_runs(n, d, ell, k, steps, tag):
    out = {}
    x, y = gpc_inputs(n, d)
    runs = [("compiled", None)] + [("numpy", None)] + [("numpy", p) for p in perms(n, N_PERM)]
    its_perm, psi_perm = [], []
    for backend, perm in runs:
        load_reference(backend)
        from defcg.gpc import KernelParams, laplace_newton, rbf_kernel
        from defcg.solvers import SolverConfig

        xs, ys = (x, y) if perm is None else (x[perm], y[perm])
        t0 = time.time()
        kmat = rbf_kernel(xs, KernelParams(1.0, ell))
        _, recs = laplace_newton(kmat, ys, "defcg", SolverConfig(tol=1e-8, ell=k + 4), newton_tol=-np.inf,
                                 max_newton=steps, k=k, selection="largest")
        del kmat
        its = np.array([r.solver_iterations for r in recs])
        psi = np.array([r.psi for r in recs])
        print(f"{tag} {backend} perm={perm is not None} its={its.tolist()} psi={psi.tolist()} "
              f"({time.time() - t0:.0f} s)", flush=True)
        if perm is None:
            b = "c" if backend == "compiled" else "n"
            out[f"{b}_its"] = its
            out[f"{b}_psi"] = psi
            out[f"{b}_rel"] = np.array([r.rel_residual for r in recs])
            out[f"{b}_f1"] = recs[0].f
        else:
            its_perm.append(its)
            psi_perm.append(psi)
    out["perm_its"] = np.array(its_perm)
    out["perm_psi"] = np.array(psi_perm)
    out["perm_idx_seed"] = np.array([12345, N_PERM])
    out["meta"] = np.array([n, d, ell, k, steps])
    return out


def config3():
    np.savez_compressed(OUT / "config3_ref.npz", **gpc_runs(24_000, 8, 2.0, 32, 3, "config3"))


def config5():
    np.savez_compressed(OUT / "config5_ref.npz", **gpc_runs(16_000, 16, 3.0, 32, 3, "config5"))


def config4(n=30_000, n_theta=3):
    x, y = sweep_inputs(n)
    thetas = np.logspace(np.log10(0.5), np.log10(2.0), 20)[:n_theta]
    out = {"thetas": thetas}
    its_perm, xerr = [], []
    runs = [None] + perms(n, 2)
    for perm in runs:
        load_reference("numpy")
        from defcg.gpc import KernelParams, rbf_kernel
        from defcg.recycle import SequenceState, solve_next
        from defcg.solvers import SolverConfig

        xs, ys = (x, y) if perm is None else (x[perm], y[perm])
        st = SequenceState(k=24, cfg=SolverConfig(tol=1e-8, ell=28), selection="largest")
        its, sols = [], []
        t0 = time.time()
        for th in thetas:
            amat = rbf_kernel(xs, KernelParams(1.0, float(th)), jitter=0.01)
            sol, st = solve_next(st, amat, ys)
            del amat
            its.append(st.history[-1].iterations)
            sols.append(sol)
            print(f"config4 perm={perm is not None} theta={th:.4f} its={its[-1]} ({time.time() - t0:.0f} s)",
                  flush=True)
        if perm is None:
            out["its"] = np.array(its)
            out["x"] = np.array(sols)
        else:
            its_perm.append(its)
            # the reference's own solution spread: the permuted run's
            # solutions mapped back to the original point order
            xs_back = np.empty_like(np.array(sols))
            xs_back[:, perm] = np.array(sols)
            xerr.append([np.linalg.norm(xb - x0) / np.linalg.norm(x0) for xb, x0 in zip(xs_back, out["x"])])
    out["perm_its"] = np.array(its_perm)
    out["perm_xerr"] = np.array(xerr)
    out["meta"] = np.array([n, 8, 24, 28])
    # the first lengthscale's system re-solved at rtol 1e-12 (the 1e-9
    # solution bar, SURVEY section 7 hard part 1(b))
    load_reference("numpy")
    from defcg.gpc import KernelParams, rbf_kernel
    from defcg.solvers import SolverConfig, cg_solve

    amat = rbf_kernel(x, KernelParams(1.0, float(thetas[0])), jitter=0.01)
    t0 = time.time()
    xt, rep, _ = cg_solve(amat, y, None, SolverConfig(tol=1e-12, ell=1))
    del amat
    print(f"config4 tight its={rep.iterations} ({time.time() - t0:.0f} s)", flush=True)
    out["tight_x"] = xt
    out["tight_its"] = np.array(rep.iterations)
    np.savez_compressed(OUT / "config4_ref.npz", **out)


def config2tight():
    out = {}
    for tag, (n, d, ell) in {"c2": (10_000, 10, 1.5), "c3": (24_000, 8, 2.0)}.items():
        load_reference("compiled")
        from defcg.gpc import KernelParams, build_newton_system, make_state, rbf_kernel
        from defcg.solvers import SolverConfig, cg_solve

        x, y = gpc_inputs(n, d)
        kmat = rbf_kernel(x, KernelParams(1.0, ell))
        sysm = build_newton_system(make_state(kmat, y))
        del kmat
        load_reference("numpy")
        from defcg.solvers import SolverConfig, cg_solve  # noqa: F811
        t0 = time.time()
        xsol, rep, _ = cg_solve(sysm.a_matrix, sysm.b, None, SolverConfig(tol=1e-12, ell=1))
        print(f"tight {tag} its={rep.iterations} rel={rep.residual_history[-1]} ({time.time() - t0:.0f} s)", flush=True)
        out[f"{tag}_x"] = xsol
        out[f"{tag}_its"] = np.array(rep.iterations)
        out[f"{tag}_meta"] = np.array([n, d, ell])
    np.savez_compressed(OUT / "config2_tight_ref.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for name, fn in [("config2tight", config2tight), ("config5", config5), ("config3", config3),
                     ("config4", config4)]:
        if which in (name, "all"):
            fn()
