#!/usr/bin/env python
"""Per-CUDA-source-line executed warp instructions of one kernel in an ncu report (cuda,sass view).
usage: ncu_lines.py REP KERNEL_INDEX [TOP]"""
import csv, io, subprocess, sys, collections


def lines(rep, k):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = collections.Counter()
    kidx, fname, hdr = -1, None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r[0] == "Function Name":
            pass
        elif r[0] == "Line No":
            hdr = r
        elif r[0] == "Kernel Name" or (len(r) > 1 and r[0] == "File Name"):
            pass
        elif hdr and r[0].isdigit() and len(r) == len(hdr):
            try:
                agg[(fname, int(r[0]))] += float(r[hdr.index("Instructions Executed")] or 0)
            except ValueError:
                pass
    return agg


def main():
    rep, k = sys.argv[1], int(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    agg = lines(rep, k)
    tot = sum(agg.values())
    print(f"total {tot:.0f}")
    for (f, ln), v in agg.most_common(top):
        print(f"{f}:{ln} {v:.0f} {v / tot * 100:.1f}%")


if __name__ == "__main__":
    main()
