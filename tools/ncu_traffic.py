#!/usr/bin/env python
"""DRAM traffic per pattern pass of one captured batched search launch (ncu --set full).
usage: ncu_traffic.py REP PATTERNS_IN_LAUNCH TEXT_BYTES OUT_JSON
The bench reads OUT_JSON (profiles/traffic_c2.json) for its roofline.traffic key."""
import csv, json, subprocess, sys

rep, P, n, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                      text=True).stdout.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
r = data[0]


def val(name):
    i = hdr.index(name)
    v = float(r[i].replace(",", ""))
    u = units[i]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(u, 1)


rd, wr, t = val("dram__bytes_read.sum"), val("dram__bytes_write.sum"), val("gpu__time_duration.sum")
res = {"kernel": r[hdr.index("Kernel Name")][:80], "patterns_in_launch": P, "text_bytes": n,
       "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_per_pattern_pass": (rd + wr) / P,
       "traffic_over_algorithmic": (rd + wr) / P / n, "duration_s_under_ncu": t,
       "source": rep.split("/")[-1] + " (ncu --set full --clock-control none, one launch)"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
