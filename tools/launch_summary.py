"""Aggregate an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])
per kernel: launches, total time, total DRAM bytes.  Development aid.

    python tools/launch_summary.py launches.csv [top]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["Kernel Name"][:90]
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg[k][0] += 1
            agg[k][1] += v
        elif d["Metric Name"].startswith("dram__bytes"):
            agg[k][2] += v
    tot = sum(a[1] for a in agg.values())
    for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{c:5d} {t / 1e3:11.1f} us {100 * t / tot:5.1f}% {b / 1e6:10.1f} MB  {k}")


if __name__ == "__main__":
    main()
