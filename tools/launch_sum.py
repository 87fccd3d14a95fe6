#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: launches, share of GPU time, avg per kernel."""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        name = r[kn].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[mv].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | share of GPU time | avg µs |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {v[0]} | {v[1] / tot * 100:.2f} % | {v[1] / v[0] / 1000:.1f} |")


if __name__ == "__main__":
    main()
