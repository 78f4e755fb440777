#!/usr/bin/env python
"""Summarise an `ncu -i rep --page source --csv --print-source cuda,sass`
export: per CUDA source line, warp-stall samples and instructions executed
(summed over its SASS), top lines first.  usage: src_hot.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
agg = {}
cur = None
for r in rows:
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        cur = (int(r[0]), r[1].strip()[:90])
        agg.setdefault(cur, [0, 0])
        continue
    if cur is None:
        continue
    d = dict(zip(hdr, r))
    try:
        agg[cur][0] += int(d["Warp Stall Sampling (All Samples)"] or 0)
        agg[cur][1] += int(d["Instructions Executed"] or 0)
    except ValueError:
        pass
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for (ln, src), (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:5d} {100*s/tot_s:5.1f}% samp {100*i/tot_i:5.1f}% inst  {src}")
