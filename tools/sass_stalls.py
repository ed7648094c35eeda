"""Stall reasons per SASS instruction of an ncu source CSV (dev tool).

usage: python tools/sass_stalls.py FILE.csv MIN_SAMPLES [LO HI]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
mn = int(sys.argv[2]) if len(sys.argv) > 2 else 300
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 1 << 30)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: 0 for r in reasons}
for i, r in enumerate(rows[2:]):
    if r and r[0] == "Kernel Name":
        break
    if len(r) < len(hdr) or not r[ix["Instructions Executed"]].isdigit():
        continue
    for k in reasons:
        tot[k] += int(r[ix[k]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    if s >= mn and lo <= i <= hi:
        top = sorted(((int(r[ix[k]] or 0), k[6:]) for k in reasons), reverse=True)[:3]
        print(f"{i:5d} {int(r[ix['Instructions Executed']]):11,d} {s:6d} {r[ix['Source']].strip()[:48]:48s} {top}")
print({k[6:]: v for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v})
