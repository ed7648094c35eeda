"""Per-kernel average of an ncu --metrics gpu__time_duration.sum --csv launch list (dev tool).

usage: python tools/launch_table.py LAUNCHES.csv
"""
import collections
import csv
import sys

d = collections.defaultdict(list)
with open(sys.argv[1]) as f:
    for r in csv.DictReader(line for line in f if line.startswith('"')):
        d[r["Kernel Name"][:48]].append(float(r["Metric Value"]))
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:50s} n={len(v):3d} avg={sum(v) / len(v) / 1e3:9.1f} us")
