#!/usr/bin/env python
"""The harmonic-Ritz pencil kernel alone on a real config-2 pencil (T = 36,
k = 16): device time per launch (CUDA events over repeated launches), the
phase stamps of the last launch, and a fingerprint of its outputs (theta, U,
active) so a rewrite can be checked bit for bit.

  python tools/pencil_bench.py [reps] [save.npz | --check ref.npz]
"""
import ctypes
import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pencil_inputs():
    import torch

    import paper_1706_00241_b200 as P
    from paper_1706_00241_b200 import gpc as G
    from paper_1706_00241_b200.recycle import harmonic_ritz_extract, refresh_basis
    from paper_1706_00241_b200.workloads import gpc_inputs

    x, y = gpc_inputs(10000, 10, 0)
    gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.5))
    st = G.make_state(gram, torch.from_numpy(y).cuda())
    sysm = G.build_newton_system(st)
    cfg = P.SolverConfig(tol=1e-8, ell=20)
    x0, _, log = P.cg_solve(sysm.a_matrix, sysm.b, None, cfg)
    ext = harmonic_ritz_extract(log, None, 16, selection="largest")
    basis = refresh_basis(sysm.a_matrix, ext.w_next_dev)
    g = torch.Generator(device="cuda").manual_seed(7)
    b2 = torch.randn(sysm.b.shape[0], dtype=torch.float64, device="cuda", generator=g)
    _, _, log2 = P.deflated_cg_solve(sysm.a_matrix, b2, x0, basis, cfg)
    m = log2.m
    W, AW = basis.w_dev, basis.aw_dev
    Pm = log2.p_dev[:m].T
    R = log2.r_dev
    al = log2.alpha_dev[:m]
    APm = ((R[:m] - R[1:m + 1]) / al[:, None]).T
    Z = torch.cat([W, Pm], 1)
    AZ = torch.cat([AW, APm], 1)
    nz = torch.linalg.norm(Z, dim=0)
    Zs, AZs = Z / nz, AZ / nz
    F = (AZs.T @ AZs).contiguous()
    Gm = (Zs.T @ AZs).contiguous()
    return F, Gm


def main():
    import torch

    from paper_1706_00241_b200 import _native as N

    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    if len(sys.argv) > 3 and sys.argv[2] == "--check":
        ref = np.load(sys.argv[3])
        F = torch.from_numpy(ref["F"]).cuda()
        Gm = torch.from_numpy(ref["G"]).cuda()
    else:
        F, Gm = pencil_inputs()
    T, k = F.shape[0], 16
    dev = F.device
    wk = torch.empty(5 * T * T, dtype=torch.float64, device=dev)
    theta = torch.empty(k, dtype=torch.float64, device=dev)
    U = torch.empty(T * k, dtype=torch.float64, device=dev)
    active = torch.empty(T, dtype=torch.int32, device=dev)
    st = torch.zeros(8, dtype=torch.int64, device=dev)
    fn = N.lib().dcg_debug_ritz_pencil
    fn.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3 + [ctypes.c_void_p] * 5
    stream = torch.cuda.current_stream().cuda_stream

    def launch():
        rc = fn(stream, F.data_ptr(), Gm.data_ptr(), T, k, 1, wk.data_ptr(), theta.data_ptr(), U.data_ptr(),
                active.data_ptr(), st.data_ptr())
        assert rc == 0, rc

    for _ in range(5):
        launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        launch()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    h = (ctypes.c_longlong * 16)()
    N.lib().dcg_debug_pencil_profile(h)
    t = list(h)
    ph = {"chol": (t[1] - t[0]) / 1e3, "C": (t[2] - t[1]) / 1e3, "tridiag": (t[8] - t[2]) / 1e3,
          "bisect": (t[9] - t[8]) / 1e3, "vectors": (t[10] - t[9]) / 1e3, "back": (t[11] - t[10]) / 1e3,
          "tail": (t[4] - t[3]) / 1e3, "total": (t[4] - t[0]) / 1e3}
    out = {"theta": theta.cpu().numpy(), "U": U.cpu().numpy(), "active": active.cpu().numpy(),
           "status": st.cpu().numpy()}
    hsh = hashlib.sha256(b"".join(np.ascontiguousarray(v).tobytes() for v in out.values())).hexdigest()[:24]
    print(f"T={T} k={k} us/launch={us:.1f} fast={t[14]} phases(us)=" +
          " ".join(f"{a}:{b:.1f}" for a, b in ph.items()) + f" sha={hsh}")
    if len(sys.argv) > 2:
        if sys.argv[2] == "--check":
            ref = np.load(sys.argv[3])
            same = all(np.array_equal(ref[a], out[a]) for a in out)
            print("bitwise identical to", sys.argv[3], ":", same)
            if not same:
                for a in out:
                    if not np.array_equal(ref[a], out[a]):
                        print("  differs:", a, np.max(np.abs(ref[a].astype(float) - out[a].astype(float))))
        else:
            np.savez(sys.argv[2], F=F.cpu().numpy(), G=Gm.cpu().numpy(), **out)


if __name__ == "__main__":
    main()
