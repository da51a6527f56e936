#!/usr/bin/env python
"""Summarise an ncu report: key throughput metrics + top stall sources (SASS)."""
import csv, io, subprocess, sys

def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout

def details(rep):
    r = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = r[0]; out = {}
    for row in r[1:]:
        d = dict(zip(h, row)); out[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    return out

def raw(rep):
    r = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    return dict(zip(r[0], r[2]))

def top_sass(rep, n=25):
    r = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    for i, row in enumerate(r):
        if row and row[0] == "Address":
            h = row; start = i; break
    i_s = h.index("Warp Stall Sampling (All Samples)"); i_src = h.index("Source"); i_ex = h.index("Instructions Executed")
    rows = []
    for row in r[start + 1:]:
        try: rows.append((int(row[i_s]), row[i_src].strip(), int(row[i_ex])))
        except Exception: pass
    tot = sum(x[0] for x in rows) or 1
    return [(s, 100.0 * s / tot, ex, src) for s, src, ex in sorted(rows, reverse=True)[:n]], sum(x[2] for x in rows)

if __name__ == "__main__":
    rep = sys.argv[1]
    d = details(rep)
    keys = ["Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "Memory Throughput",
            "L2 Hit Rate", "Issued Ipc Active", "Achieved Active Warps Per SM", "Registers Per Thread",
            "Dynamic Shared Memory Per Block", "No Eligible", "Executed Instructions"]
    for k in keys:
        if k in d: print(f"{k:36s} {d[k][0]} {d[k][1]}")
    rw = raw(rep)
    for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__cycles_active.min", "sm__cycles_active.max",
              "lts__t_bytes.sum", "l1tex__t_bytes.sum"]:
        if k in rw: print(f"{k:60s} {rw[k]}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(v)) for k, v in rw.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    print("stalls:", ", ".join(f"{k}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
    if "--sass" in sys.argv:
        rows, tot = top_sass(rep)
        print("instructions executed:", tot)
        for s, pct, ex, src in rows:
            print(f"{s:7d} {pct:5.1f}% ex={ex:9d} {src[:95]}")
