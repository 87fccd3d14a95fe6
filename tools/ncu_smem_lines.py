#!/usr/bin/env python
"""Shared-memory wavefronts per CUDA source line of an ncu report (--import-source on): which
lines carry the excessive (bank-conflicted) wavefronts.  usage: ncu_smem_lines.py REP [TOP]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, fname = None, "?"
tot = collections.Counter()
exc = collections.Counter()
text = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
        iw, ie, isrc = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive"), hdr.index("Source")
    elif hdr and r[0].isdigit() and len(r) == len(hdr):
        try:
            w, e = float(r[iw] or 0), float(r[ie] or 0)
        except ValueError:
            continue
        key = (fname, int(r[0]))
        tot[key] += w
        exc[key] += e
        text.setdefault(key, r[isrc].strip()[:100])
W, E = sum(tot.values()), sum(exc.values())
print(f"shared wavefronts {W:.3e}, excessive {E:.3e} ({100 * E / max(W, 1):.1f} %)")
print("| line | wavefronts | excessive | share of all excessive | source |")
print("|---|---|---|---|---|")
for key, e in exc.most_common(top):
    print(f"| {key[0]}:{key[1]} | {tot[key]:.3e} | {e:.3e} | {100 * e / max(E, 1):.1f} % | `{text[key]}` |")
