#!/usr/bin/env python
"""Executed instructions / stall samples of one ncu capture grouped by source function
(line ranges of the CURRENT search_impl.cuh: capture and source must match).
usage: ncu_funcs.py REP"""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = hdr = None
ie, st = collections.Counter(), collections.Counter()
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit():
        try:
            ie[(fname, int(r[0]))] += float(r[hdr.index("Instructions Executed")] or 0)
            st[(fname, int(r[0]))] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            pass
src = open("paper_1612_01506_b200/csrc/search_impl.cuh").read().split("\n")
starts = []
for i, l in enumerate(src):
    m = re.match(r"(?:__device__|__global__|template|struct)\b.*?\b(\w+)\s*\(", l) if not l.startswith(" ") else None
    m2 = re.match(r"^(?:__device__ __forceinline__|__device__|__global__ void).*?(\w+)\(", l)
    if m2:
        starts.append((i + 1, m2.group(1)))
def func(ln):
    name = "?"
    for a, n in starts:
        if a <= ln:
            name = n
    return name
I, S = sum(ie.values()), sum(st.values())
agg, ags = collections.Counter(), collections.Counter()
for (f, ln), v in ie.items():
    key = func(ln) if f == "search_impl.cuh" else f
    agg[key] += v
    ags[key] += st[(f, ln)]
for k, v in agg.most_common(20):
    print(f"{k:28s} {v / I * 100:5.1f}% instr {ags[k] / S * 100:5.1f}% stalls")
