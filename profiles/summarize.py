"""Summaries of ncu output for profiles/ (run here on the merged gpurun_out/ files).

  python profiles/summarize.py launches <launches.csv>            -> per-kernel table
  python profiles/summarize.py full <report.ncu-rep>              -> key metrics of the captured launch
  python profiles/summarize.py fullall <report.ncu-rep>           -> the same for every captured launch
  python profiles/summarize.py traffic <report.ncu-rep> n mv k its -> solve_kernel_dram.json payload
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path):
    rows = [l for l in open(path) if l.startswith('"')]
    r = list(csv.reader(rows))
    h = r[0]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for row in r[1:]:
        d = per[int(row[iid])]
        d[row[im]] = float(row[iv].replace(",", ""))
        d["name"] = row[ik].split("(")[0].replace("void ", "")[:60]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        a = agg[d["name"]]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':60s} {'launches':>8s} {'ms':>9s} {'share%':>7s} {'DRAM GB/s':>10s}"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:60s} {v[0]:8d} {v[1] / 1e6:9.3f} {100 * v[1] / tot:7.1f} {v[2] / v[1] if v[1] else 0:10.1f}")
    out.append(f"total {tot / 1e6:.3f} ms over {len(per)} launches (ncu: cold caches, serialised)")
    return "\n".join(out)


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    return r[0], r[1], r[2]


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
]


def full(rep):
    h, u, v = raw(rep)
    out = []
    for k in KEYS:
        if k in h:
            i = h.index(k)
            out.append(f"{k:70s} {v[i]:>16s} {u[i]}")
    return "\n".join(out)


def fullall(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, u = r[0], r[1]
    out = []
    for v in r[2:]:
        out.append("== " + v[h.index("Kernel Name")].split("(")[0])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"{k:70s} {v[i]:>16s} {u[i]}")
    return "\n".join(out)


def traffic(rep, n, mv, k, its):
    h, u, v = raw(rep)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rb = float(v[h.index("dram__bytes_read.sum")]) * scale[u[h.index("dram__bytes_read.sum")]]
    wb = float(v[h.index("dram__bytes_write.sum")]) * scale[u[h.index("dram__bytes_write.sum")]]
    n, mv, k, its = int(n), int(mv), int(k), int(its)
    alg = mv * 8 * n * (n + 1) // 2 + 8 * n * (2 * k + 10) * its
    return json.dumps({"n": n, "k": k, "iterations": its, "matvec_equivalents": mv, "dram_bytes": rb + wb,
                       "dram_read": rb, "dram_write": wb, "alg_bytes": alg, "traffic_over_alg": (rb + wb) / alg,
                       "source": rep}, indent=1)


if __name__ == "__main__":
    mode = sys.argv[1]
    print({"launches": launches, "full": full, "fullall": fullall, "traffic": traffic}[mode](*sys.argv[2:]))
