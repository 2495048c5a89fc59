"""A W block-product time (the refresh's product) through the public operator:
packed symmetric DMMA product vs the row-major DMMA GEMM.
  python tools/block_probe.py [n] [k] [reps]"""
import json, os, sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1706_00241_b200 as P  # noqa: E402
from paper_1706_00241_b200.workloads import gpc_inputs  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
x, _ = gpc_inputs(n, 10)
gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.5))
s = torch.rand(n, dtype=torch.float64, device="cuda") * 0.5
w = torch.randn(n, k, dtype=torch.float64, device="cuda")
out = {"n": n, "k": k}
for strat in ("sym", "rows"):
    A = gram.scaled(s, 1.0).with_strategy(strat)
    for _ in range(3):
        y = A.apply_block_dev(w)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        y = A.apply_block_dev(w)
    e1.record()
    torch.cuda.synchronize()
    out[strat + "_us"] = e0.elapsed_time(e1) * 1e3 / reps
    out[strat + "_sum"] = float(y.sum())
print(json.dumps(out))
