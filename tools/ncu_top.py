#!/usr/bin/env python
"""Summarise an ncu source page: top SASS lines / CUDA lines by executed instructions and stall samples."""
import csv
import io
import subprocess
import sys


def page(rep, view, kernel_idx=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name"')
    blk = blocks[1 + kernel_idx]
    lines = blk.split("\n", 1)[1]
    rows = list(csv.reader(io.StringIO(lines)))
    hdr = rows[0]
    return hdr, rows[1:]


def main():
    rep = sys.argv[1]
    view = sys.argv[2] if len(sys.argv) > 2 else "sass"
    k = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    hdr, rows = page(rep, view, k)
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    src = hdr.index("Source")
    tot_i = sum(float(r[ie] or 0) for r in rows if len(r) > ie)
    tot_s = sum(float(r[ss] or 0) for r in rows if len(r) > ss)
    print(f"total instructions {tot_i:.0f}  stall samples {tot_s:.0f}")
    rows = [r for r in rows if len(r) > max(ie, ss)]
    if view == "sass":
        for r in rows:
            pass
    srt = sorted(rows, key=lambda r: -float(r[ss] or 0))[:top]
    for r in srt:
        print(f"{float(r[ss] or 0)/max(tot_s,1)*100:5.1f}%S {float(r[ie] or 0)/max(tot_i,1)*100:5.1f}%I  {r[0][-6:]:>6} {r[src].strip()[:110]}")


if __name__ == "__main__":
    main()
