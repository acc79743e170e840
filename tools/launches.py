"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: mean us per kernel."""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
ix = {k: j for j, k in enumerate(rows[h])}
d = OrderedDict()
for r in rows[h + 1:]:
    if len(r) < len(rows[h]) or r[ix['Metric Name']] != 'gpu__time_duration.sum':
        continue
    name = r[ix['Kernel Name']].split('(')[0]
    v = float(r[ix['Metric Value']].replace(',', ''))
    unit = r[ix['Metric Unit']]
    v = v / 1000.0 if unit in ('nsecond', 'ns') else (v * 1000.0 if unit in ('msecond', 'ms') else v)
    d.setdefault(name, []).append(v)
tot = 0.0
for k, v in d.items():
    m = sum(v) / len(v); tot += m
    print(f"{k:40s} n={len(v):3d} mean {m:9.2f} us")
print(f"{'sum of means':40s}       {tot:9.2f} us")
