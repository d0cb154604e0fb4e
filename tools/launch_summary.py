"""Summarise an ncu --metrics gpu__time_duration.sum CSV log per kernel (tools helper)."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d['Metric Name'] != 'gpu__time_duration.sum': continue
        v = float(d['Metric Value'].replace(',', '')); u = d['Metric Unit']
        v = v / 1e3 if u in ('nsecond', 'ns') else (v * 1e3 if u in ('msecond', 'ms') else v)
        k = d['Kernel Name'].split('(')[0][-48:]
        agg[k][0] += 1; agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:10.1f} us {v[0]:5d} launches {v[1]/v[0]:9.1f} us/launch {100*v[1]/tot:5.1f}%  {k}")
print(f"total {tot:.1f} us")
