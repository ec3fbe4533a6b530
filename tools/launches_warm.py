"""Summarise an ncu launch list with gpu__time_duration.sum (+ optional lts__t_bytes.sum,
dram__bytes_read.sum) per kernel.  python tools/launches_warm.py LIST.csv [iterations]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
iters = float(sys.argv[2]) if len(sys.argv) > 2 else 11
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[h]
ki, mi, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].split('::')[-1]
    if '<' in r[ki]:
        name += r[ki][r[ki].index('<'):r[ki].index('>') + 1]
    v = float(r[vi].replace(',', ''))
    if r[mi] == 'gpu__time_duration.sum':
        v = {'ns': v / 1000, 'nsecond': v / 1000, 'ms': v * 1000, 'msecond': v * 1000}.get(r[ui], v)
    agg[name][r[mi]].append(v)
tot = sum(sum(m['gpu__time_duration.sum']) for m in agg.values())
for k, m in sorted(agg.items(), key=lambda kv: -sum(kv[1]['gpu__time_duration.sum'])):
    t = m['gpu__time_duration.sum']
    extra = ""
    for key, lab in (('lts__t_bytes.sum', 'L2'), ('dram__bytes_read.sum', 'dram')):
        if m.get(key):
            extra += f"  {lab} {sum(m[key]) / len(m[key]) / 1e6:6.2f} MB"
    print(f"{k[:28]:28s} n={len(t):3d} mean {sum(t) / len(t):7.2f} us  min {min(t):7.2f}  share {sum(t) / tot:5.1%}{extra}")
print(f"total {tot:.1f} us, per iteration {tot / iters:.1f} us")
