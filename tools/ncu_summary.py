"""Key metrics of every kernel in an ncu report: python tools/ncu_summary.py report.ncu-rep"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_bytes.sum"]
ix = {k: h.index(k) for k in keys if k in h}
units = rows[1]
for r in rows[2:]:
    print("----", r[ix["Kernel Name"]][:60])
    for k in keys[1:]:
        if k in ix:
            print(f"  {k:60s} {r[ix[k]]:>16s} {units[ix[k]]}")
stall = [(k, r) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
for r in rows[2:]:
    vals = sorted(((float(r[h.index(k)] or 0), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k, _ in stall), reverse=True)
    tot = sum(v for v, _ in vals) or 1
    print("  stalls:", ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in vals[:7]))
