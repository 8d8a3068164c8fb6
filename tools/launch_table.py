#!/usr/bin/env python
"""Per-launch table (duration, DRAM read/write bytes) from an ncu --csv --metrics log of one bench step
command: tools/launch_table.py <csv> <out.txt> <header line>"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
by = collections.OrderedDict()
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
         "msecond": 1e3, "nsecond": 1e-3}
for d in data:
    k = (int(d["ID"]), d["Kernel Name"].split("(")[0])
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1)
    by.setdefault(k, {})[d["Metric Name"]] = v
with open(sys.argv[2], "w") as f:
    f.write(sys.argv[3].rstrip() + "\n")
    f.write(f"{'id':>3s} {'kernel':58s} {'us':>10s} {'DRAM rd MB':>11s} {'DRAM wr MB':>11s} {'GB/s':>8s}\n")
    tot = collections.Counter()
    for (i, n), m in by.items():
        us = m.get("gpu__time_duration.sum", 0.0)
        rd = m.get("dram__bytes_read.sum", 0.0) / 1e6
        wr = m.get("dram__bytes_write.sum", 0.0) / 1e6
        f.write(f"{i:3d} {n[:58]:58s} {us:10.1f} {rd:11.2f} {wr:11.2f} {(rd + wr) * 1e3 / max(us, 1e-9):8.0f}\n")
print(open(sys.argv[2]).read())
