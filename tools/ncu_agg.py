"""Aggregate an ncu --csv launch list (metrics per launch) by kernel name + grid:
count, mean duration, mean DRAM bytes.  Usage: python tools/ncu_agg.py launches.csv"""
import csv, sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
launches = OrderedDict()
for r in rows[1:]:
    d = launches.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]]})
    d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
groups = OrderedDict()
prev = None
for d in launches.values():
    key = (d["name"][:60], d["grid"], round(d.get("dram__bytes_read.sum", 0) / 64e6))
    # consecutive runs of the same kernel form a group
    if prev is None or prev[0] != key:
        groups[len(groups)] = (key, [])
        prev = groups[len(groups) - 1]
    prev[1].append(d)
for key, ds in groups.values():
    n = len(ds)
    avg = lambda m: sum(x.get(m, 0.0) for x in ds) / n
    print(f"{key[0]:60s} {key[1]:>14s} x{n:<3d} {avg('gpu__time_duration.sum')/1e3:9.1f} us  "
          f"rd {avg('dram__bytes_read.sum')/1e6:8.1f} MB  wr {avg('dram__bytes_write.sum')/1e6:7.1f} MB")
