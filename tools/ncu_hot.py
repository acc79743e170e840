"""Print the hottest SASS instructions (by warp-stall samples) of an ncu report, with a
window of surrounding instructions.  Usage: python tools/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[1:]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
order = sorted(range(len(data)), key=lambda i: -int(data[i][ix["Warp Stall Sampling (All Samples)"]] or 0))
print(f"total samples {tot}, instructions {len(data)}")
for i in order[:n]:
    r = data[i]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{100.0*s/tot:5.1f}% #{i:5d} exec={r[ix['Instructions Executed']]:>9} {r[ix['Source']].strip()}")
