"""Per-kernel summary of an ncu --metrics launch list (CSV log):
kernel, launches, total device ms, time share, ms per launch, DRAM GB read /
written per launch, warp instructions per launch.
usage: python scripts/launch_summary.py LAUNCHES.csv > SUMMARY.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
h = rows[0]
ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
per = defaultdict(dict)
for r in rows[1:]:
    if len(r) < len(h):
        continue
    key = (r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", ""))
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    name = r[ix["Metric Name"]]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
             "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(unit, 1.0)
    per[key][name] = v * scale
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
for (_, k), m in per.items():
    a = agg[k]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
    a[4] += m.get("smsp__inst_executed.sum", 0.0)
tot = sum(a[1] for a in agg.values()) or 1.0
w = csv.writer(sys.stdout)
w.writerow(["kernel", "launches", "total_ms", "share", "avg_ms", "dram_read_GB_per_launch",
            "dram_write_GB_per_launch", "warp_inst_per_launch"])
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    n = a[0]
    w.writerow([k, n, round(a[1], 3), round(a[1] / tot, 4), round(a[1] / n, 4), round(a[2] / n, 4),
                round(a[3] / n, 4), int(a[4] / n)])
