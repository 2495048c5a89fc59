import sys, ctypes, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_1706_00241_b200 as P
from paper_1706_00241_b200 import _native as N, recycle
from paper_1706_00241_b200.workloads import gpc_inputs
x, y = gpc_inputs(10000, 10, 0)
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.5))
yd = torch.from_numpy(y).cuda()
cfg = P.SolverConfig(tol=1e-8, ell=20)
orig = recycle._AsyncSolve.finish
def fin(job):
    out = orig(job)
    if job.pending is not None:
        job.pending.join(torch.cuda.current_stream())
        job.pending.event.synchronize()
        h = (ctypes.c_longlong * 16)()
        N.lib().dcg_debug_pencil_profile.restype = ctypes.c_int
        N.lib().dcg_debug_pencil_profile(h)
        t = list(h)
        print(f"pencil T-after-prune={t[6]} sweeps={t[7]} chol/prune={(t[1]-t[0])/1e3:.1f}us  gchol+B={(t[2]-t[1])/1e3:.1f}us jacobi={(t[3]-t[2])/1e3:.1f}us tail={(t[4]-t[3])/1e3:.1f}us total={(t[4]-t[0])/1e3:.1f}us fast={t[14]} [tridiag {(t[8]-t[2])/1e3:.1f} bisect {(t[9]-t[8])/1e3:.1f} invit {(t[10]-t[9])/1e3:.1f} back {(t[11]-t[10])/1e3:.1f} cyc/count {t[12]/max(t[13],1):.0f} its {t[13]}] rounds={t[13]} cyc/round load={t[8]/max(t[13],1):.0f} shfl={t[9]/max(t[13],1):.0f} rot={t[10]/max(t[13],1):.0f} upd={t[11]/max(t[13],1):.0f} bar={t[12]/max(t[13],1):.0f}")
    return out
recycle._AsyncSolve.finish = fin
P.laplace_newton(gram, yd, "defcg", cfg, newton_tol=-np.inf, max_newton=8, k=16, selection="largest")
