# K7 (matrix-free pass 1): timing, then one ncu capture with the pipe / stall metrics of profiles/r02/k7_*_ncu.txt
mkdir -p gpurun_out
timeout 120 python tools/k7_probe.py 50000 16 6 | tee gpurun_out/k7_probe.json
timeout 120 python tools/k7_probe.py 30000 16 6 | tee -a gpurun_out/k7_probe.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rbf_mma_pass1_kernel -s 2 -c 1 -o gpurun_out/k7_full -f python tools/k7_probe.py 30000 16 2 > gpurun_out/k7_ncu.log 2>&1
ncu -i gpurun_out/k7_full.ncu-rep --page raw --csv > gpurun_out/k7_raw.csv 2>/dev/null
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/k7_raw.csv")))
hdr, val = rows[0], rows[-1]
want = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__inst_executed.avg.per_cycle_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
for h, v in zip(hdr, val):
    if h in want or h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
        try:
            if float(v.replace(",", "")) >= 0.1 or h in want: print(f"{h:85s} {v}")
        except ValueError:
            pass
PY
