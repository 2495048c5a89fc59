import os, sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1706_00241_b200 as P
from oracle.defcg_oracle import gpc_inputs
n = int(sys.argv[1])
x, y = gpc_inputs(n, 8, 0)
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 2.0))
st0 = P.gpc.make_state(gram, torch.from_numpy(y).cuda())
sys0 = P.gpc.build_newton_system(st0)
os.environ["DCG_PHASE_TIMERS"] = "1"
P.cg_solve(sys0.a_matrix, sys0.b, torch.zeros(n, dtype=torch.float64, device="cuda"), P.SolverConfig(tol=1e-8, ell=0))
import ctypes
buf = (ctypes.c_ulonglong * 1024)()
P._native.lib().dcg_debug_phase_timers_all(buf, 1024)
G = 148
p2 = [buf[16 + G + b] / 1e3 for b in range(G)]
p1 = [buf[16 + b] / 1e3 for b in range(G)]
print("pass2 per-CTA (us total):", " ".join(f"{v:.0f}" for v in p2))
print("pass1 per-CTA (us total):", " ".join(f"{v:.0f}" for v in p1[::8]))
