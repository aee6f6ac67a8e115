"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py gpurun_out/r9/launches_cfg5.csv
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path):
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        us = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
        name = d["Kernel Name"].replace("void ", "").split("(")[0]
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':58s} {'launches':>8s} {'total_ms':>9s} {'per_launch_us':>13s} {'share':>6s}")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:58]:58s} {n:8d} {us / 1e3:9.3f} {us / n:13.1f} {100 * us / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
