#!/usr/bin/env python3
"""Stall-reason summary of an ncu source-page CSV (ncu -i X --page source --csv --print-source sass):
totals per stall reason, and the top SASS instructions by samples with their dominant reason."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r][0]
hdr, data = rows[hi], rows[hi + 1:]
src = hdr.index("Source")
smp = hdr.index("Warp Stall Sampling (All Samples)")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
lines = []
for r in data:
    if len(r) <= smp or not r[smp].isdigit():
        continue
    per = {hdr[i]: int(r[i] or 0) for i in cols if r[i].isdigit()}
    tot.update(per)
    lines.append((int(r[smp]), r[0][-5:], r[src].strip()[:70], max(per, key=per.get) if per else ""))
T = sum(tot.values())
print("total samples", T)
for k, v in tot.most_common(12):
    print(f"  {k:24s} {v:7d} {100 * v / T:5.1f}%")
print("top instructions:")
for n, a, s, why in sorted(lines, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"  {n:6d} {a} {why:22s} {s}")
