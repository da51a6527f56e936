#!/usr/bin/env python
"""Warp-stall samples of an ncu report aggregated by source line (file:line, inlined code
attributed to its own file) and the top stalled SASS instructions with context.
Usage: python tools/stall_lines.py REPORT.ncu-rep [n]"""
import csv, io, subprocess, sys

def page(rep, what):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", what],
                         capture_output=True, text=True, cwd="/tmp").stdout
    return list(csv.reader(io.StringIO(out)))

def main():
    import os; rep = os.path.abspath(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    rows = page(rep, "cuda,sass")
    f = cur = None; agg = {}
    for r in rows:
        if r and r[0] == "File Path": f = r[1].split("/")[-1]; continue
        if len(r) < 5: continue
        if r[0].strip(): cur = (f, r[0], r[1].strip()[:80])
        try: s = int(r[4])
        except ValueError: continue
        agg[cur] = agg.get(cur, 0) + s
    tot = sum(agg.values()) or 1
    print(f"total stall samples {tot}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
        print(f"{v:6d} {100*v/tot:5.1f}% {k[0]}:{k[1]} {k[2]}")
    rows = page(rep, "sass")
    for i, r in enumerate(rows):
        if r and r[0] == "Address": h = r; st = i; break
    iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    body = rows[st + 1:]
    tops = sorted(range(len(body)), key=lambda i: -int(body[i][iW] or 0))[:8]
    for t in sorted(tops):
        print("-----")
        for j in range(max(0, t - 4), min(len(body), t + 2)):
            r = body[j]
            print(">>" if j == t else "  ", r[0][-5:], r[iW].rjust(6), r[iE].rjust(8), r[iS])

main()
