"""Standalone K v product time (the public operator's symmetric product).
  python tools/matvec_probe.py [n] [reps]"""
import json, os, sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
x, _ = gpc_inputs(n, 10)
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.5)).kernel_view()
v = torch.randn(n, dtype=torch.float64, device="cuda")
y = gram.matvec_dev(v)
for _ in range(5):
    gram.matvec_dev(v, out=y)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(reps):
    gram.matvec_dev(v, out=y)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
print(json.dumps({"n": n, "us_per_product": us, "GBps": 8 * n * (n + 1) / 2 / (us * 1e-6) / 1e9,
                  "lib": os.environ.get("DCG_LIB_PATH"), "checksum": float(y.sum())}))
