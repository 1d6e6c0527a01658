#!/usr/bin/env python3
"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch):
total time and launch count per kernel, largest first.
usage: launch_summary.py launches.csv [divide_by]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    agg[r[ki][:80]][0] += 1
    agg[r[ki][:80]][1] += v
tot = sum(v for _, v in agg.values())
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c / div:7.2f} {v / 1e3 / div:10.1f} us {100 * v / tot:5.1f}%  {k}")
print(f"total {tot / 1e3 / div:.1f} us per unit")
