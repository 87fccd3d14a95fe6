#!/usr/bin/env python
"""NEXT-2: the paper's order comparison (Tables 1-4 columns N32 / N32-freq / N32-fixed,
PAPER.md:201-331) on B200: device GB/s per (config, m, order, strategy).

Orders: identity (Algs. 1-2), pi_h / pi_hs (fixed), freq (rarest
first from the text histogram).  Strategies: BLOCK with the
paper's peeling factor r = 2 (freq) / 3 (others), and FILTER."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1612_01506_b200 as sm
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c2,c3,c1")
ap.add_argument("--n", type=int, default=1 << 28)
ap.add_argument("--lengths", default="4,8,16,32,64")
ap.add_argument("--per-m", type=int, default=8)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
torch.cuda.set_device(0)
d = torch.zeros(1, dtype=torch.int64, device="cuda")
for cfg in a.configs.split(","):
    spec = synth.text_spec(cfg, n=a.n)
    t = synth.gen_text_device(spec, 0, spec.n)
    hist = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
    lengths = [int(x) for x in a.lengths.split(",")]
    pats = synth.patterns(cfg, spec=spec, per_m=a.per_m, lengths=lengths)
    for m in lengths:
        ps = [p.data for p in pats if p.m == m and p.kind == "sampled"]
        row = {"cfg": cfg, "m": m}
        for oname in ("identity", "pi_h", "pi_hs", "freq"):
            orders = [None if oname == "freq" else
                      sm.sm_heuristic_order(p, {"identity": 0, "pi_h": 1, "pi_hs": 2}[oname]) for p in ps]
            for sname, strat, peel in (("block", 2, 2 if oname == "freq" else 3), ("filter", 1, 0)):
                def run():
                    for p, o in zip(ps, orders):
                        sm.sm_count_async(p, t, d, hist=hist, order=o, strategy=strat, peel=peel)
                run()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.reps):
                    run()
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / (a.reps * len(ps))
                row[f"{sname}/{oname}"] = round(spec.n / us / 1e3, 1)
        print(json.dumps(row), flush=True)
    del t
    torch.cuda.empty_cache()
