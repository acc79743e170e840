"""Executed instructions and stall samples per CUDA source line of an ncu report (cuda,sass
view; needs -lineinfo): python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
ex = collections.Counter()
st = collections.Counter()
src = {}
fname = ""
h = None
cur = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = {k: i for i, k in enumerate(r)}
        ie = r.index("Instructions Executed")
        isamp = r.index("Warp Stall Sampling (All Samples)")
        continue
    if h is None or len(r) < 4:
        continue
    if r[0]:  # a CUDA source line row
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:100]
    if cur is None:
        continue
    try:
        ex[cur] += int(r[ie] or 0)
        st[cur] += int(r[isamp] or 0)
    except (ValueError, IndexError):
        pass
tex = sum(ex.values()) or 1
tst = sum(st.values()) or 1
print(f"total executed {tex}, stall samples {tst}")
for k, v in ex.most_common(top):
    print(f"{100.0 * v / tex:5.1f}% exec {100.0 * st[k] / tst:5.1f}% stall  {k[0]}:{k[1]:<5} {src.get(k, '')}")
print("-- by stall samples")
for k, v in st.most_common(top // 2):
    print(f"{100.0 * ex[k] / tex:5.1f}% exec {100.0 * v / tst:5.1f}% stall  {k[0]}:{k[1]:<5} {src.get(k, '')}")
