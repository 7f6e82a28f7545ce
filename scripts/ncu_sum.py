#!/usr/bin/env python3
"""Sum an ncu --metrics gpu__time_duration.sum CSV per kernel: python scripts/ncu_sum.py f.csv [top]"""
import collections
import csv
import sys

t = collections.defaultdict(float)
n = collections.Counter()
for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')):
    if r["Metric Name"] == "gpu__time_duration.sum":
        k = r["Kernel Name"][:70]
        t[k] += float(r["Metric Value"].replace(",", ""))
        n[k] += 1
tot = sum(t.values())
for k, v in sorted(t.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{v / 1e3:10.1f} us {100 * v / tot:5.1f}%  {n[k]:5d}  {k}")
