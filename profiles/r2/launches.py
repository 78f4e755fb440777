#!/usr/bin/env python
"""Print an ncu launch list (--metrics gpu__time_duration.sum --csv) as
id / kernel / microseconds, plus the total.  usage: launches.py file.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = 0.0
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            us = v / 1e3 if d["Metric Unit"] == "ns" else (v if d["Metric Unit"] == "us" else v * 1e3)
            tot += us
            print(f"{d['ID']:>4} {us:10.2f} us  {d['Kernel Name'][:90]}")
print(f"total {tot:.1f} us")
