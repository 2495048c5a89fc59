"""Diagnostic: def-CG at config 3's recipe (k = 32, ell_log = 36), n = 24,000.

Runs the first Newton system's plain-CG solve on the GPU, then the harmonic
Ritz extraction of its log on the GPU and in the oracle (same log), and
compares Ritz values and the spans; then the first 3 Newton steps with the
pencil's tridiagonal fast path on and off.
  python tools/diag_config3.py [n]"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from oracle import defcg_oracle as O  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24_000
k, ell = 32, 36
x, y = gpc_inputs(n, 8)
gram = P.rbf_kernel(x, P.KernelParams(1.0, 2.0))
st = P.gpc.make_state(gram, y)
sysm = P.gpc.build_newton_system(st)
xs, rep, log = P.cg_solve(sysm.a_matrix, sysm.b, None, P.SolverConfig(tol=1e-8, ell=ell))
print("first solve its", rep.iterations, "stored", log.stored_iterations, flush=True)
out = {}
olog = O.Log(d=list(log.d), alpha=list(log.alpha), beta=list(log.beta), mu=[], p=[np.asarray(v) for v in log.p],
             r=[np.asarray(v) for v in log.r])
# F and its pivots from the GPU's log, in numpy
m = len(olog.p)
z = np.stack(olog.p, 1)
az = np.stack([(olog.r[j] - olog.r[j + 1]) / olog.alpha[j] for j in range(m)], 1)
nrm = np.linalg.norm(z, axis=0)
z, az = z / nrm, az / nrm
F = az.T @ z
F = 0.5 * (F + F.T)
print("F eig range", np.linalg.eigvalsh(F)[[0, -1]], "diag range", np.diag(F).min(), np.diag(F).max())
print("alpha", np.array(olog.alpha)[:5], "... d", np.array(olog.d)[:3])
try:
    L, fail = O.backend("numpy").cholesky(F, 1e-14 * np.max(np.diag(F)))
    print("numpy-F cholesky fail index", fail)
except Exception as e:
    print("chol err", e)
for fast in (1, 0):
    P._native.lib().dcg_debug_set_pencil_fast(fast)
    try:
        ext = P.harmonic_ritz_extract(log, None, k, "largest")
        out[fast] = ext
        print("gpu fast", fast, "theta[:5]", np.asarray(ext.theta.cpu())[:5])
    except Exception as e:
        print("gpu fast", fast, "raised", repr(e))
P._native.lib().dcg_debug_set_pencil_fast(1)
oext = O.harmonic_ritz(olog, None, k, "largest", be="numpy")
print("oracle theta[:5]", oext.theta[:5], "theta[-3:]", oext.theta[-3:])


def proj(w):
    q, _ = np.linalg.qr(w)
    return q


qo = proj(oext.w_next)
for fast, ext in out.items():
    th = ext.theta.cpu().numpy()
    wg = ext.w_next.cpu().numpy()
    qg = proj(wg)
    s = np.linalg.svd(qo.T @ qg, compute_uv=False)
    print(f"fast={fast}: max |theta - oracle| rel {np.max(np.abs(th - oext.theta) / np.abs(oext.theta)):.3e}; "
          f"principal-angle cosines min {s.min():.6f}; W norms {np.linalg.norm(wg, axis=0).min():.3e}")
    # W'AW conditioning
    aw = ext.aw_next.cpu().numpy()
    gmat = wg.T @ aw
    ev = np.linalg.eigvalsh(0.5 * (gmat + gmat.T))
    print(f"   W'AW eigen range {ev.min():.3e} .. {ev.max():.3e}")
for fast in (1, 0):
    P._native.lib().dcg_debug_set_pencil_fast(fast)
    _, recs = P.laplace_newton(gram, y, "defcg", P.SolverConfig(tol=1e-8, ell=ell), newton_tol=-np.inf,
                               max_newton=3, k=k, selection="largest")
    print("newton its fast", fast, [r.solver_iterations for r in recs], flush=True)
P._native.lib().dcg_debug_set_pencil_fast(1)
# the non-pipelined sequence (solve_next on explicit Newton systems)
seq = P.SequenceState(k=k, cfg=P.SolverConfig(tol=1e-8, ell=ell), selection="largest")
state = P.gpc.make_state(gram, y)
its = []
for it in range(3):
    sm = P.gpc.build_newton_system(state)
    xs, seq = P.solve_next(seq, sm.a_matrix, sm.b)
    its.append(seq.history[-1].iterations)
    state, _ = P.gpc._update_dev(state, sm.inner, sm.sqrt_h, xs if isinstance(xs, torch.Tensor) else torch.from_numpy(xs).cuda())
print("solve_next (sync) its", its)
np.savez_compressed("gpurun_out/log24k.npz", p=np.stack(olog.p), r=np.stack(olog.r), alpha=np.array(olog.alpha),
                    d=np.array(olog.d), beta=np.array(olog.beta))
