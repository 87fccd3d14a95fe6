#!/usr/bin/env python
"""Dump per-SASS-instruction executed counts (percent of total) and stall samples from an ncu report."""
import csv, io, subprocess, sys
rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
blk = out.split('"Kernel Name"')[1 + k].split("\n", 1)[1]
rows = list(csv.reader(io.StringIO(blk)))
hdr = rows[0]; rows = [r for r in rows[1:] if len(r) == len(hdr)]
ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)"); te = hdr.index("Thread Instructions Executed")
ti = sum(float(r[ie]) for r in rows); ts = sum(float(r[ss]) for r in rows) or 1
print(f"# total warp instructions {ti:.0f}, samples {ts:.0f}")
for r in rows:
    f = float(r[ie]) / ti * 100
    print(f"{r[0][-5:]} {f:6.3f} S{float(r[ss])/ts*100:5.2f} {float(r[te])/max(float(r[ie]),1):5.1f} {r[1].strip()[:100]}")
