import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests/golden')
from oracle import defcg_oracle as O

def prune_trace(p, r, alpha, be="numpy"):
    m = p.shape[0]
    z = p.T.copy(); az = np.stack([(r[j] - r[j + 1]) / alpha[j] for j in range(m)], 1)
    nrm = np.linalg.norm(z, axis=0); z /= nrm; az /= nrm
    dropped = []
    idx = list(range(m))
    while True:
        f = az.T @ z; f = 0.5 * (f + f.T)
        L, fail = O.backend(be).cholesky(f, 1e-14 * np.max(np.diag(f)))
        if fail < 0: break
        dropped.append(idx[fail]); del idx[fail]
        z = np.delete(z, fail, 1); az = np.delete(az, fail, 1)
    return dropped

g = np.load('gpurun_out/log24k.npz  (written by tools/diag_config3.py on the GPU box)')
#print("GPU log: dropped", prune_trace(g['p'], g['r'], g['alpha']))
print("GPU log alpha[:8]", g['alpha'][:8])
# the reference's own log of the same first system
from make_golden import load_reference, gpc_inputs
load_reference("numpy")
from defcg.gpc import KernelParams, build_newton_system, make_state, rbf_kernel
from defcg.solvers import SolverConfig, cg_solve
x, y = gpc_inputs(24000, 8)
K = rbf_kernel(x, KernelParams(1.0, 2.0))
sysm = build_newton_system(make_state(K, y))
del K
xs, rep, log = cg_solve(sysm.a_matrix, sysm.b, None, SolverConfig(tol=1e-8, ell=36))
print("ref its", rep.iterations)
p = np.array(log.p); r = np.array(log.r); al = np.array(log.alpha)
#print("REF log: dropped", prune_trace(p, r, al))
print("ref alpha[:8]", al[:8])
print("p diff vs gpu (rel, first 8):", [float(np.linalg.norm(p[j]-g['p'][j])/np.linalg.norm(p[j])) for j in range(0,36,5)])

def conj(p, r, alpha):
    m = p.shape[0]
    z = p.T.copy(); az = np.stack([(r[j] - r[j + 1]) / alpha[j] for j in range(m)], 1)
    f = az.T @ z; f = 0.5 * (f + f.T)
    dg = np.sqrt(np.abs(np.diag(f)))
    c = np.abs(f) / np.outer(dg, dg)
    np.fill_diagonal(c, 0)
    return [float(c[j, :j].max()) if j else 0.0 for j in range(m)]
cg = conj(g['p'], g['r'], g['alpha']); cr = conj(p, r, al)
print("max |cos_A(p_j, p_i<j)|   j: gpu / ref")
for j in range(0, 36, 3): print(f"  {j:2d}: {cg[j]:.2e} / {cr[j]:.2e}")
# residual orthogonality
def rorth(r):
    rn = r / np.linalg.norm(r, axis=1)[:, None]
    c = np.abs(rn @ rn.T); np.fill_diagonal(c, 0)
    return [float(c[j, :j].max()) if j else 0 for j in range(r.shape[0])]
og = rorth(g['r']); orf = rorth(r)
print("max |cos(r_j, r_i<j)|")
for j in range(0, 37, 3): print(f"  {j:2d}: {og[j]:.2e} / {orf[j]:.2e}")
