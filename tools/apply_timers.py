"""Per-CTA phases of the standalone symmetric product (DCG_APPLY_TIMERS=1):
set-up, pass 1, grid barrier, pass 2, relative to the earliest CTA start (us)."""
import ctypes, os, sys
os.environ["DCG_APPLY_TIMERS"] = "1"
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200 import _native as N  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
x, _ = gpc_inputs(n, 10)
k = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.5)).kernel_view()
v = torch.randn(n, dtype=torch.float64, device="cuda")
for _ in range(5):
    k.matvec_dev(v)
torch.cuda.synchronize()
G = 147
buf = (ctypes.c_ulonglong * (5 * G))()
lib = N.lib()
lib.dcg_debug_apply_timers.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert lib.dcg_debug_apply_timers(buf, 5 * G) == 0
t = np.array(buf, dtype=np.float64).reshape(G, 5)
t0 = t[:, 0].min()
t = (t - t0) / 1e3
for name, col in (("start", 0), ("setup_done", 1), ("pass1_done", 2), ("barrier_done", 3), ("end", 4)):
    print(f"{name:14s} min {t[:, col].min():7.2f} mean {t[:, col].mean():7.2f} max {t[:, col].max():7.2f}")
d1 = t[:, 2] - t[:, 1]
print("pass1 per CTA (us):", " ".join(f"{v:.0f}" for v in d1))
