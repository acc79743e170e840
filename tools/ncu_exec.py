"""Aggregate executed warp-instructions of an ncu report by SASS region (window of W
instructions) to find where the instruction budget goes.  Usage: ncu_exec.py rep [W] [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; W = int(sys.argv[2]) if len(sys.argv) > 2 else 200; N = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
h = rows[0]; ix = {k: i for i, k in enumerate(h)}; data = rows[1:]
ex = [int(r[ix["Instructions Executed"]] or 0) for r in data]
tot = sum(ex)
print(f"total warp-inst {tot:,}")
wins = [(sum(ex[i:i + W]), i) for i in range(0, len(ex), W)]
wins.sort(reverse=True)
for s, i in wins[:N]:
    top = max(range(i, min(i + W, len(ex))), key=lambda j: ex[j])
    print(f"{100.0*s/tot:5.1f}%  [{i:6d}..{i+W:6d})  hottest #{top} x{ex[top]:,}: {data[top][ix['Source']].strip()[:70]}")
