"""DRAM traffic per corpus pass of a kernel family, from an ncu launch list
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
over `bench.py --profile-run`, i.e. ONE complete run), into
profiles/traffic.json (bench.py's roofline.traffic).

  python scripts/traffic_from_launches.py CSV CONFIG PASSES [FAMILY=regex ...]
"""
import csv
import json
import os
import re
import sys

FAMILIES = {"count_all": r"k_count_(all|hot)<", "route_scatter": r"k_route_scatter",
            "route_consume": r"k_consume", "route_count": r"k_route_count",
            "once_direct": r"k_once_direct"}


def main():
    path, cfg, passes = sys.argv[1], sys.argv[2], int(sys.argv[3])
    fams = dict(FAMILIES)
    for a in sys.argv[4:]:
        k, v = a.split("=", 1)
        fams[k] = v
    hdr, per = None, {}
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "byte")
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        for f, rx in fams.items():
            if re.search(rx, d["Kernel Name"]):
                per[f] = per.get(f, 0.0) + v
    out_p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                         "profiles", "traffic.json")
    tj = json.load(open(out_p)) if os.path.exists(out_p) else {}
    for f, v in per.items():
        tj[f"{cfg}:{f}"] = v / passes
        print(f"{cfg}:{f}", round(v / passes / 1e9, 3), "GB per corpus pass")
    tj.setdefault("_sources", {})[cfg] = (f"{os.path.basename(path)}: dram__bytes_read.sum + "
                                          f"dram__bytes_write.sum of one bench.py --profile-run, "
                                          f"summed per family / {passes} corpus passes")
    json.dump(tj, open(out_p, "w"), indent=1)


if __name__ == "__main__":
    main()
