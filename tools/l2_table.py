"""Per-kernel duration / DRAM bytes / L2 hit rate table from an ncu --csv metrics log.
python tools/l2_table.py LOG.csv"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[h]
ki, mi, vi, ui, idi = (hdr.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
d = OrderedDict()
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    d.setdefault((r[idi], r[ki].split('(')[0][-34:]), {})[r[mi]] = (r[vi], r[ui])
for (i, k), m in d.items():
    g = lambda n: m.get(n, ('-', ''))
    print(f"{i:>4} {k:34s} t={g('gpu__time_duration.sum')[0]:>8}{g('gpu__time_duration.sum')[1]:4s} "
          f"dramR={g('dram__bytes_read.sum')[0]:>9}{g('dram__bytes_read.sum')[1]:6s} "
          f"hit={g('lts__t_sector_hit_rate.pct')[0]}")
