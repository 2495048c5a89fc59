#!/usr/bin/env python
"""GPU timeline of one config-2 Newton sequence (torch.profiler / CUPTI
activity records: real concurrent timings, unlike ncu's serialised replay).

  python tools/timeline.py [n] [out.json]

Prints per-kernel totals, the busy/idle split of the main stream and the
per-Newton-step critical-path segments; writes the raw event list as JSON.
"""
import collections
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_1706_00241_b200 as P
    from paper_1706_00241_b200.workloads import gpc_inputs

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/timeline.json"
    # config 2 (n = 10k: d 10, l 1.5, k 16) or config 3 (n = 50k: d 8, l 2, k 32)
    d, ell, k = (8, 2.0, 32) if n >= 50000 else (10, 1.5, 16)
    x, y = gpc_inputs(n, d, 0)
    gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, ell))
    yd = torch.from_numpy(y).cuda()
    cfg = P.SolverConfig(tol=1e-8, ell=k + 4)

    def run():
        return P.laplace_newton(gram, yd, "defcg", cfg, newton_tol=-np.inf, max_newton=8, k=k, selection="largest")

    for _ in range(1 if n >= 50000 else 3):
        run()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        run()
        torch.cuda.synchronize()
    evs = []
    for e in prof.events():
        if e.device_type.name == "CUDA" and e.time_range.elapsed_us() >= 0:
            evs.append({"name": e.name, "start": e.time_range.start, "end": e.time_range.end,
                        "stream": getattr(e, "device_resource_id", None) or getattr(e, "stream", None)})
    evs.sort(key=lambda d: d["start"])
    t0 = evs[0]["start"]
    t1 = max(d["end"] for d in evs)
    Path(out).parent.mkdir(parents=True, exist_ok=True)
    Path(out).write_text(json.dumps(evs))
    tot = collections.defaultdict(float)
    for d in evs:
        tot[d["name"][:60]] += d["end"] - d["start"]
    print(f"span {t1 - t0:.1f} us, {len(evs)} device events")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
        print(f"  {v:9.1f} us  {k}")
    # union of busy intervals (any stream)
    busy, cur_s, cur_e = 0.0, None, None
    for d in evs:
        if cur_e is None or d["start"] > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = d["start"], d["end"]
        else:
            cur_e = max(cur_e, d["end"])
    busy += cur_e - cur_s
    print(f"device busy (any stream) {busy:.1f} us = {100 * busy / (t1 - t0):.1f}% of span")
    # listing: start offset, duration, gap to previous end, name
    print("timeline (us from start: start dur gap name)")
    prev_end = t0
    for d in evs:
        gap = d["start"] - prev_end
        print(f"  {d['start'] - t0:9.1f} {d['end'] - d['start']:8.1f} {gap:7.1f}  s{d['stream']}  {d['name'][:70]}")
        prev_end = max(prev_end, d["end"])


if __name__ == "__main__":
    main()
