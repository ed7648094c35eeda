"""Hottest SASS instructions of an ncu --page source --print-source sass CSV (dev tool).

usage: python tools/sass_hot.py FILE.csv [N]   (prints the N top instructions by
executed count and by stall samples, plus the total)
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
recs = []
for i, r in enumerate(rows[2:]):
    if r and r[0] == "Kernel Name":
        break  # first kernel section only
    if len(r) < len(hdr) or not r[ix["Instructions Executed"]].isdigit():
        continue
    recs.append((i, r[ix["Source"]].strip(), int(r[ix["Instructions Executed"]] or 0),
                 int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
tot = sum(x[2] for x in recs)
stall = sum(x[3] for x in recs)
print(f"total warp instructions {tot:,}  stall samples {stall:,}")
for i, src, ex, st in recs:
    if ex > tot * 0.004 or st > stall * 0.01:
        print(f"{i:5d} {ex:12,d} {st:7d}  {src}")
