"""Attribute ncu per-SASS executed instructions / stall samples to CUDA source lines using
nvdisasm line info.  Usage: ncu_lines.py report.ncu-rep lib.so kernel_substring [N]"""
import csv, io, re, subprocess, sys, tempfile, os, glob, collections
rep, so, kname = sys.argv[1], sys.argv[2], sys.argv[3]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
h = rows[0]; ix = {k: i for i, k in enumerate(h)}; data = rows[1:]
ex = [int(r[ix["Instructions Executed"]] or 0) for r in data]
st = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = glob.glob(os.path.join(d, "*.cubin"))[0]
sass = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout.splitlines()
# find section of the kernel
start = None
for i, l in enumerate(sass):
    if l.startswith("//----") and kname in l:
        start = i; break
lines = []
cur = ("?", 0)
for l in sass[start + 1:]:
    if l.startswith("//----"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        lines.append(cur)
print(f"sass instr in ncu: {len(data)}, in nvdisasm: {len(lines)}")
agg_e = collections.Counter(); agg_s = collections.Counter()
for i in range(min(len(lines), len(data))):
    agg_e[lines[i]] += ex[i]; agg_s[lines[i]] += st[i]
te, ts = sum(ex), sum(st)
print("by executed instructions:")
for k, v in agg_e.most_common(N):
    print(f"  {100.0*v/te:5.1f}% exec  {100.0*agg_s[k]/ts:5.1f}% stall  {k[0]}:{k[1]}")
print("by stall samples:")
for k, v in agg_s.most_common(N):
    print(f"  {100.0*v/ts:5.1f}% stall {100.0*agg_e[k]/te:5.1f}% exec  {k[0]}:{k[1]}")
