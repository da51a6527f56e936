#!/usr/bin/env python
"""Turn one round's ncu captures (tools/profile_round.sh) into the tracked summaries:

    profiles/<tag>_launches.csv      per-launch gpu__time_duration of two forward steps
    profiles/<tag>_kernels.md        per-launch table from the --set full capture of one step
    profiles/ncu_traffic.json        per stage group: mean DRAM bytes per launch (bench.py's
                                     roofline.traffic) + the launch durations they came from

Usage: python tools/profile_summary.py TAG [gpurun_out]
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_csv(path):
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def stage_of(name, index_in_step, pruned_seen):
    name = name[5:] if name.startswith("void ") else name
    if name.startswith("k_tokenize"):
        return "tokenizer"
    if name.startswith("k_head") or "GsHead" in name:
        return "head"
    if name.startswith("k_gather_rows"):
        return "gather"
    if "k_attention" in name:
        return "attention"
    if "k_block_tail" in name:
        return "tail"
    if "EpiQKVG" in name:
        return "qkvg"
    if "EpiSwiGLU" in name:
        return "ffn_up"
    if "EpiResid" in name:
        return "wo|ffn_down"
    return name.split("(")[0]


def label_steps(names):
    """Assign stage labels; EpiResid alternates wo -> ffn_down inside each layer."""
    out, resid = [], 0
    for n in names:
        s = stage_of(n, 0, False)
        if s == "wo|ffn_down":
            s = "wo" if resid % 2 == 0 else "ffn_down"
            resid += 1
        out.append(s)
    return out


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)

    # ---- launch list
    rows = read_csv(os.path.join(src, f"launches_{tag}.csv"))
    h = rows[0]
    iN, iV, iG = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    launches = [(r[iN], r[iG], float(r[iV]) / 1e3) for r in rows[1:]]
    with open(os.path.join(prof, f"{tag}_launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["launch", "stage", "kernel", "grid", "gpu_time_us"])
        labels = label_steps([l[0] for l in launches])
        for i, ((n, g, t), s) in enumerate(zip(launches, labels)):
            w.writerow([i, s, n.split("(")[0], g, f"{t:.2f}"])

    # ---- full capture (one step)
    rows = read_csv(os.path.join(src, f"full_{tag}_raw.csv"))
    h = rows[0]
    units, data = rows[1], rows[2:]  # row 1 holds units
    scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def col(r, name, conv=float):
        """Value in base units (ns, bytes) -- the raw page picks a unit per column."""
        try:
            i = h.index(name)
            v = conv(r[i].replace(",", ""))
            return v * scale[units[i]] if conv is float and units[i] in scale else v
        except (ValueError, IndexError):
            return None

    names = [r[h.index("Kernel Name")] for r in data]
    labels = label_steps(names)
    recs = []
    for r, s in zip(data, labels):
        dur_ns = col(r, "gpu__time_duration.sum")
        rd = col(r, "dram__bytes_read.sum")
        wr = col(r, "dram__bytes_write.sum")
        rec = {
            "stage": s, "kernel": r[h.index("Kernel Name")].split("(")[0],
            "grid": r[h.index("Grid Size")], "block": r[h.index("Block Size")],
            "us": dur_ns / 1e3 if dur_ns else None,
            "dram_read": rd, "dram_write": wr,
            "dram_pct": col(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "tensor_pct": col(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
            or col(r, "sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "sm_pct": col(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            "regs": col(r, "launch__registers_per_thread", int),
            "ipc": col(r, "sm__inst_executed.avg.per_cycle_active"),
        }
        recs.append(rec)
    tot_us = sum(r["us"] or 0 for r in recs)

    def fmt(v, f="{:.1f}"):
        return "-" if v is None else f.format(v)

    lines = [f"# ncu --set full, one SORT-base forward step ({tag})", "",
             "Captured by `tools/profile_round.sh` (`ncu --set full --clock-control none`, one",
             "step after 3 warm-up steps; per-launch times are serialised and cold-cache, so",
             "compare SHARES with bench.py's stage breakdown, not absolutes).", "",
             "| # | stage | kernel | grid | us | share | DRAM rd MB | DRAM wr MB | DRAM % | tensor % | SM % | IPC | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for i, r in enumerate(recs):
        lines.append(
            f"| {i} | {r['stage']} | `{r['kernel'][:40]}` | {r['grid']} | {fmt(r['us'])} | "
            f"{fmt(100 * (r['us'] or 0) / tot_us)}% | {fmt((r['dram_read'] or 0) / 1e6)} | "
            f"{fmt((r['dram_write'] or 0) / 1e6)} | {fmt(r['dram_pct'])} | {fmt(r['tensor_pct'])} | "
            f"{fmt(r['sm_pct'])} | {fmt(r['ipc'], '{:.2f}')} | {r['regs']} |")
    lines += ["", f"Total (serialised) {tot_us:.1f} us.", ""]
    groups = {}
    for r in recs:
        g = groups.setdefault(r["stage"], {"launches": 0, "us": 0.0, "bytes": 0.0})
        g["launches"] += 1
        g["us"] += r["us"] or 0
        g["bytes"] += (r["dram_read"] or 0) + (r["dram_write"] or 0)
    lines += ["| stage | launches | us | share | DRAM bytes / launch |", "|---|---|---|---|---|"]
    traffic = {"tag": tag, "source": f"profiles/{tag}_kernels.md (ncu --set full, one step)",
               "unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum), mean"}
    for s, g in sorted(groups.items(), key=lambda kv: -kv[1]["us"]):
        per = g["bytes"] / g["launches"]
        traffic[s] = per
        lines.append(f"| {s} | {g['launches']} | {g['us']:.1f} | {100 * g['us'] / tot_us:.1f}% | "
                     f"{per / 1e6:.1f} MB |")
    open(os.path.join(prof, f"{tag}_kernels.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(os.path.join(prof, "ncu_traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
