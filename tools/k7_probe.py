"""Matrix-free product (K7) alone: python tools/k7_probe.py [n] [d] [reps] -> ms per product, contract-model fraction."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 16
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((n, d))).cuda()
op = P.rbf_kernel(x, P.KernelParams(1.0, 3.0), matrix_free=True)
v = torch.from_numpy(rng.standard_normal(n)).cuda()
y = op.matvec_dev(v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(reps):
    e0.record(); op.matvec_dev(v, out=y); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
flop = float(n) * (n + 1) / 2 * (2 * d + 4)
print(json.dumps({"n": n, "d": d, "ms": best, "tflops_contract": flop / best / 1e9, "frac_dmma_peak": flop / best / 1e9 / 37.1,
                  "checksum": float(y.sum())}))
