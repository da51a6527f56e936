"""Aggregate an ncu `--metrics gpu__time_duration.sum --csv` launch list per kernel.

usage: python tools/launch_agg.py launches.csv [steps_captured] [top]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[r[ki][:80]][0] += 1
        agg[r[ki][:80]][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot / 1e3 / steps:.1f} us/step over {steps:g} step(s)")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v / 1e3 / steps:9.1f} us/step {n / steps:6.1f} launches  {k}")


if __name__ == "__main__":
    main()
