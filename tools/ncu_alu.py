#!/usr/bin/env python
"""ALU-pipe work of one bench step of a compare-bound config (SURVEY.md §8(d) ALU roofline).

Two modes:
  python tools/ncu_alu.py run CONFIG        -- one sm_count_batch of the config's full pattern set
                                               (the bench step's search launches); run it under
        ncu --metrics smsp__inst_executed_pipe_alu.sum,smsp__inst_executed.sum,gpu__time_duration.sum,
                      sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,
                      smsp__issue_active.avg.pct_of_peak_sustained_active
            -k regex:search_kernel --csv --log-file X.csv
  python tools/ncu_alu.py sum X.csv CONFIG OUT_JSON  -- sums the search launches into OUT_JSON
        (profiles/alu_<config>.json), which bench.py reads for roofline.achieved in ALU
        warp-instructions per step.

Instruction counts do not depend on timing, so the counts from the (serialised,
cold-cache) ncu replay divided by the bench's live search time give the achieved rate.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(config):
    import numpy as np
    import torch

    import paper_1612_01506_b200 as sm
    import synth
    torch.cuda.set_device(0)
    spec = synth.text_spec(config)
    t = synth.gen_text_device(spec, 0, spec.n)
    pats = synth.patterns(config, spec=spec)
    hist = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch([p.data for p in pats], t, d, hist=hist)
    torch.cuda.synchronize()
    print(json.dumps({"config": config, "patterns": len(pats), "count_sum": int(d.sum().item())}))


def summarise(csv_path, config, out):
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    per = {}
    for r in rows[1:]:
        if "search_kernel" not in r[ix["Kernel Name"]]:
            continue
        k = int(r[ix["ID"]])
        v = float(r[ix["Metric Value"]].replace(",", ""))
        u = r[ix["Metric Unit"]]
        if r[ix["Metric Name"]] == "gpu__time_duration.sum":
            v *= {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(u, 1)
        per.setdefault(k, {"kernel": r[ix["Kernel Name"]][:90]})[r[ix["Metric Name"]]] = v
    launches = list(per.values())
    tot = lambda key: sum(x.get(key, 0.0) for x in launches)
    import synth
    res = {
        "config": config,
        "patterns": len(synth.patterns(config)),
        "text_bytes": synth.text_spec(config).n,
        "launches": len(launches),
        "alu_warp_inst_per_step": tot("smsp__inst_executed_pipe_alu.sum"),
        "warp_inst_per_step": tot("smsp__inst_executed.sum"),
        "search_s_under_ncu": tot("gpu__time_duration.sum"),
        "alu_pipe_active_pct": [round(x.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 0), 1)
                                for x in launches],
        "issue_active_pct": [round(x.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0), 1)
                             for x in launches],
        "kernels": sorted({x["kernel"] for x in launches}),
        "source": os.path.basename(csv_path) + " (ncu --clock-control none, every search launch of one "
                  "sm_count_batch over the config's full pattern set)",
    }
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        summarise(sys.argv[2], sys.argv[3], sys.argv[4])
