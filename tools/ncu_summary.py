"""One line per captured launch of `ncu --set full` reports: duration, DRAM and L2 bytes,
achieved DRAM bandwidth, fp64 pipe activity, warps active, launch shape.
python tools/ncu_summary.py REPORT.ncu-rep [...] > summary.csv"""
import csv
import subprocess
import sys

KEYS = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"), ("lts__t_bytes.sum", "l2_bytes"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_pct"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
        ("TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "fp64_pipe_pct"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "regs")]
SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
w = csv.writer(sys.stdout)
w.writerow(["report"] + [k for _, k in KEYS] + ["dram_GBps"])
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        vals = []
        for key, _ in KEYS:
            if key not in hdr:
                vals.append("")
                continue
            i = hdr.index(key)
            v = r[i].replace(",", "")
            try:
                v = float(v) * SCALE.get(units[i], 1.0)
                v = round(v, 3)
            except ValueError:
                v = v.split("(")[0][:40]
            vals.append(v)
        try:
            gbps = round((vals[2] + vals[3]) / (vals[1] * 1e-6) / 1e9, 1)
        except (TypeError, ZeroDivisionError):
            gbps = ""
        w.writerow([rep.split("/")[-1]] + vals + [gbps])
