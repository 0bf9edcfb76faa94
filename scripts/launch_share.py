"""Summarise an ncu --metrics gpu__time_duration.sum launch list (per-kernel share)."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[vi].replace(',', ''))
    except ValueError:
        continue
    agg[r[ki].split('(')[0]][0] += 1
    agg[r[ki].split('(')[0]][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:70]:70s} launches={v[0]:3d} total={v[1]/1e6:10.3f} ms share={v[1]/tot*100:5.1f}%")
