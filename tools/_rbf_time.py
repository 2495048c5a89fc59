"""Time the stored RBF Gram assembly (rbf_kernel) at config-2 size."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1706_00241_b200 as P  # noqa: E402
from oracle.defcg_oracle import gpc_inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
x, y = gpc_inputs(n, 10, 0)
xd = torch.from_numpy(x).cuda()
for _ in range(3):
    g = P.rbf_kernel(xd, P.KernelParams(1.0, 1.5))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g = P.rbf_kernel(xd, P.KernelParams(1.0, 1.5))
e1.record()
torch.cuda.synchronize()
print(f"rbf_kernel n={n}: {e0.elapsed_time(e1) / 10:.3f} ms")
kd = g.dense_dev()
print("exactly symmetric:", bool(torch.equal(kd, kd.T)))
