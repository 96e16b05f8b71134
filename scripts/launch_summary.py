#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python scripts/launch_summary.py gpurun_out/launches.csv [--skip-name REGEX]

Prints per-kernel-signature count, total and mean device time and share.
ncu serialises launches and runs them cold: compare SHARES with bench.py's
live CUDA-event numbers, not absolutes.
"""

import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                data.append(d)
    return data


def key(d):
    name = d["Kernel Name"]
    name = re.sub(r"\(mrs::\w+\)$", "", name)
    return f"{name[:80]}  grid={d['Grid Size']}"


def main():
    path = sys.argv[1]
    data = load(path)
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(data[0]["Metric Unit"], 1e-3)
    agg = collections.OrderedDict()
    for d in data:
        a = agg.setdefault(key(d), [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"].replace(",", "")) * scale
    tot = sum(a[1] for a in agg.values())
    print(f"{'count':>6} {'total_us':>10} {'mean_us':>9} {'share':>6}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:6d} {t:10.1f} {t / c:9.2f} {100 * t / tot:5.1f}%  {k}")
    print(f"launches {len(data)}  total {tot:.1f} us")


if __name__ == "__main__":
    main()
