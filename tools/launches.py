"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[h]; data = rows[h + 1:]
ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = defaultdict(list)
for r in data[skip:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].split('::')[-1]
    if '<' in r[ki]:
        name += r[ki][r[ki].index('<'):r[ki].index('>') + 1]
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    us = {'ns': v / 1000, 'nsecond': v / 1000, 'us': v, 'usecond': v, 'ms': v * 1000, 'msecond': v * 1000}[u]
    agg[name].append(us)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':32s} {'n':>4s} {'mean us':>9s} {'min us':>8s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:32]:32s} {len(v):4d} {sum(v)/len(v):9.2f} {min(v):8.2f} {sum(v)/tot:6.1%}")
print(f"total {tot:.1f} us over {sum(len(v) for v in agg.values())} launches")
