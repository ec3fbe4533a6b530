"""Aggregate ncu warp-stall samples by CUDA source line (and top stall reasons).
python tools/ncu_lines.py REPORT.ncu-rep [min_share]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.008
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, src, fname = collections.Counter(), {}, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 4 and r[0].isdigit():
        try:
            c = int(r[4])
        except ValueError:
            continue
        key = (fname, int(r[0]))
        agg[key] += c
        src.setdefault(key, r[1][:100])
tot = sum(agg.values())
print("total samples", tot)
for k, c in sorted(agg.items(), key=lambda kv: (kv[0][0] or "", kv[0][1])):
    if c > tot * thr:
        print(f"{k[0]}:{k[1]:4d} {c:6d} {100 * c / tot:5.1f}%  {src[k]}")
