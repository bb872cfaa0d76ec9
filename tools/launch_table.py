#!/usr/bin/env python
"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum --csv): per kernel name the
launch count, median and last duration in us.  Dev tool."""
import collections
import csv
import statistics
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    if len(r) <= vi:
        continue
    n = r[ki].split("(")[0]
    agg.setdefault(n, []).append(float(r[vi].replace(",", "")) / 1e3)
for n, v in agg.items():
    print(f"{n[:40]:40s} n={len(v):4d} median={statistics.median(v):9.1f}us last={v[-1]:9.1f}us")
