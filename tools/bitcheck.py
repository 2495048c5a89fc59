#!/usr/bin/env python
"""Bitwise fingerprint of full def-CG Newton sequences (the pipelined GPC path).

  python tools/bitcheck.py [out.json]

Prints (and writes) a SHA-256 of the final latent f, the psi trajectory and the
iteration counts for config 1, config 2, the config-3 recipe at n = 12,000 (stored Gram)
and the config-5 recipe at n = 20,000 (matrix-free).  A refactoring that claims to keep the arithmetic
(operation order, rounding) must leave every fingerprint unchanged.
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import paper_1706_00241_b200 as P
    from paper_1706_00241_b200.workloads import CONFIGS, gpc_inputs

    out = {}
    cases = [("config1", CONFIGS[1], None), ("config2", CONFIGS[2], None), ("config3@12k", CONFIGS[3], 12000),
             ("config5@20k-mf", CONFIGS[5], 20000)]
    for name, c, nover in cases:
        n = nover or c["n"]
        x, y = gpc_inputs(n, c["d"])
        gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, c["lengthscale"]),
                            matrix_free=bool(c.get("matrix_free")))
        cfg = P.SolverConfig(tol=c["tol"], ell=c["ell"])
        st, recs = P.laplace_newton(gram, torch.from_numpy(y).cuda(), "defcg", cfg, newton_tol=-np.inf,
                                    max_newton=c["newton_steps"], k=c["k"], selection="largest")
        f = st.f.detach().cpu().numpy()
        h = hashlib.sha256(f.tobytes())
        h.update(np.array([r.psi for r in recs]).tobytes())
        out[name] = {"its": [r.solver_iterations for r in recs], "sha": h.hexdigest()[:24],
                     "psi_last": repr(recs[-1].psi)}
        print(name, out[name], flush=True)
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
