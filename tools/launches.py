#!/usr/bin/env python3
"""Summarize an ncu --csv launch list (gpu__time_duration.sum): per kernel
name, count and total microseconds.  Usage: python tools/launches.py file.csv"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    h = None
    agg = defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows:
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                k = d["Kernel Name"][:70]
                v = float(d["Metric Value"]) * (1e-3 if d.get("Metric Unit") in ("nsecond", "ns") else 1.0)
                if k not in agg:
                    order.append(k)
                agg[k][0] += 1
                agg[k][1] += v
    tot = sum(v for _, v in agg.values())
    for k in sorted(agg, key=lambda x: -agg[x][1]):
        n, v = agg[k]
        print(f"{n:4d} {v:9.2f} us  {100 * v / tot:5.1f}%  {k}")
    print(f"total {tot:.2f} us, {sum(n for n, _ in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
