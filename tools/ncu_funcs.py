"""Attribute an ncu report's executed instructions/stall samples to the functions (labels)
of the kernel's SASS.  Usage: ncu_funcs.py report lib.so kernel_mangled_substring"""
import csv, io, re, subprocess, sys, tempfile, os, glob, collections
rep, so, kname = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
h = rows[0]; ix = {k: i for i, k in enumerate(h)}; data = rows[1:]
ex = [int(r[ix["Instructions Executed"]] or 0) for r in data]
st = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = glob.glob(os.path.join(d, "*.cubin"))[0]
sass = subprocess.run(["nvdisasm", "-c", cub], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(sass) if l.startswith("//----") and kname in l)
fn = "kernel"; owner = []
for l in sass[start + 1:]:
    if l.startswith("//----"): break
    m = re.match(r"^\s*([\$\.\w]+):\s*$", l)
    if m and not m.group(1).startswith(".L_x") and not m.group(1).startswith(".text"):
        fn = m.group(1)
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        owner.append(fn)
print(len(owner), len(data))
agg = collections.Counter(); aggs = collections.Counter()
for i in range(min(len(owner), len(data))):
    agg[owner[i]] += ex[i]; aggs[owner[i]] += st[i]
te, ts = sum(ex), sum(st)
for k, v in agg.most_common(40):
    name = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    print(f"{100.0*v/te:5.1f}% exec {100.0*aggs[k]/ts:5.1f}% stall  {name[:110]}")

if len(sys.argv) > 4:
    # detail: hottest instructions (by stall samples) inside functions matching argv[4]
    pat = sys.argv[4]
    idx = [i for i in range(min(len(owner), len(data))) if pat in owner[i]]
    idx.sort(key=lambda i: -st[i])
    for i in idx[:40]:
        print(f"  #{i:6d} stall={st[i]:6d} exec={ex[i]:9d}  {data[i][ix['Source']].strip()[:90]}")
