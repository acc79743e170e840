"""SASS of one kernel in an ncu report with executed-instruction counts and stall samples,
grouped into basic-block-ish runs.  Usage: ncu_sass.py report.ncu-rep kernel_regex [top]"""
import csv, io, re, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kre, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]; ix = {k: i for i, k in enumerate(h)}
data = []
for r in rows[1:]:
    if r and r[0] == "Kernel Name":
        break  # first matching launch only
    if len(r) >= len(h) - 1:
        data.append(r)
ie, ss = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]
tot = sum(int(r[ie] or 0) for r in data); tots = sum(int(r[ss] or 0) for r in data)
print(f"total exec {tot}  samples {tots}  instrs {len(data)}")
# group consecutive instructions with equal exec count
groups = []
for i, r in enumerate(data):
    e = int(r[ie] or 0); s = int(r[ss] or 0)
    if groups and groups[-1][1] == e:
        groups[-1][2] += 1; groups[-1][3] += s; groups[-1][4].append(r[ix["Source"]].strip())
    else:
        groups.append([i, e, 1, s, [r[ix["Source"]].strip()]])
groups.sort(key=lambda g: -g[1] * g[2])
for g in groups[:top]:
    print(f"#{g[0]:5d} exec={g[1]:>9d} x{g[2]:3d} = {100*g[1]*g[2]/tot:5.1f}% exec, {100*g[3]/max(1,tots):5.1f}% stall | {' ; '.join(g[4][:4])[:150]}")
