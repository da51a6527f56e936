"""Per-kernel time and DRAM bytes of an ncu launch list captured with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv:
achieved GB/s per kernel (the row kernels of the training step are HBM-bound).
usage: python tools/train_bw.py launches.csv [steps] [top]"""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    h = rows[0]
    ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        try:
            per[(r[ii], r[ki][:70])][r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, k), m in per.items():
        a = agg[k]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot / 1e3 / steps:.1f} us/step")
    print(f"{'us/step':>9} {'n':>5} {'MB/launch':>10} {'GB/s':>7}  kernel")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t / 1e3 / steps:9.1f} {n / steps:5.1f} {b / n / 1e6:10.1f} {b / t:7.0f}  {k}")


if __name__ == "__main__":
    main()
