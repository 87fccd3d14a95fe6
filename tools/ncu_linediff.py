#!/usr/bin/env python
"""Per-source-line executed-instruction diff between two kernels of one ncu report (cuda,sass view).
usage: ncu_linediff.py REP [A_IDX B_IDX TOP]"""
import collections, csv, io, subprocess, sys


def per_kernel(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    aggs, fname, hdr, cur, lastfn = [], None, None, None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r[0] == "Function Name":
            if r[1] != lastfn:
                cur = collections.Counter()
                aggs.append(cur)
                lastfn = r[1]
        elif r[0] == "Line No":
            hdr = r
        elif hdr and r[0].isdigit():
            try:
                cur[(fname, int(r[0]))] += float(r[hdr.index("Instructions Executed")] or 0)
            except ValueError:
                pass
    return aggs


def main():
    rep = sys.argv[1]
    i, j = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 1)
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    ag = per_kernel(rep)
    a, b = ag[i], ag[j]
    print("totals", sum(a.values()), sum(b.values()))
    for k in sorted(set(a) | set(b), key=lambda k: -(b[k] - a[k]))[:top]:
        print(k, a[k], b[k], b[k] - a[k])


if __name__ == "__main__":
    main()
