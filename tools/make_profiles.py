"""Summarise ncu captures (gpurun_out/) into tracked files under profiles/.

    python tools/make_profiles.py TAG config:report.ncu-rep [config:report ...]

Writes profiles/<TAG>_<config>_ncu.txt (per kernel: duration, DRAM bytes, L2 bytes,
instructions, occupancy, issue activity, top stall reasons) and merges per-kernel DRAM
traffic per launch into profiles/ncu_traffic.json (read by bench.py for roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"), ("lts__t_bytes.sum", "l2_bytes"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
        ("smsp__inst_executed.sum", "warp_instr"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
        ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3,
         "ms": 1e3, "msecond": 1e3}


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    tag = sys.argv[1]
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for arg in sys.argv[2:]:
        cfg, rep = arg.split(":", 1)
        h, units, data = rows_of(rep)
        ix = {k: h.index(k) for k, _ in KEYS if k in h}
        stall_keys = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
        lines = [f"# ncu --set full --clock-control none, {cfg}, report {os.path.basename(rep)} "
                 f"(cold-cache, serialised replays: per-kernel SHARES are meaningful, absolute times are not bench values)"]
        per = {}
        for r in data:
            name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
            vals = {}
            for k, short in KEYS:
                if k in ix:
                    v = r[ix[k]].replace(",", "")
                    try:
                        vals[short] = float(v) * SCALE.get(units[ix[k]], 1.0)
                    except ValueError:
                        vals[short] = v
            st = sorted(((float(r[h.index(k)] or 0), k.split("stalled_")[1]) for k in stall_keys), reverse=True)
            tot = sum(v for v, _ in st) or 1.0
            vals["stalls"] = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in st[:4])
            per.setdefault(name, []).append(vals)
        tot_us = sum(v["duration"] for lst in per.values() for v in lst)
        lines.append(f"{'kernel':22s} {'us':>9s} {'share':>6s} {'DRAM rd MB':>10s} {'DRAM wr MB':>10s} {'L2 MB':>8s} "
                     f"{'Minstr':>8s} {'occ%':>5s} {'issue%':>6s}  top stalls")
        traffic.setdefault(cfg, {})
        for name, lst in per.items():
            v = lst[0]
            lines.append(f"{name:22s} {v['duration']:9.2f} {v['duration'] / tot_us:6.3f} {v['dram_read'] / 1e6:10.2f} "
                         f"{v['dram_write'] / 1e6:10.2f} {v.get('l2_bytes', 0) / 1e6:8.2f} {v['warp_instr'] / 1e6:8.2f} "
                         f"{v['occupancy_pct']:5.1f} {v['issue_active_pct']:6.1f}  {v['stalls']}")
            traffic[cfg][name] = round(v["dram_read"] + v["dram_write"])
        lines.append(f"{'sum':22s} {tot_us:9.2f}")
        out = os.path.join(ROOT, "profiles", f"{tag}_{cfg}_ncu.txt")
        open(out, "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
