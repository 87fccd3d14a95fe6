#!/usr/bin/env python
"""Per-pattern device time of FILTER vs BLOCK (several r) on a config: data for the AUTO model."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1612_01506_b200 as sm
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--lengths", default="2,3,4,6,8,16")
ap.add_argument("--per-m", type=int, default=12)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
torch.cuda.set_device(0)
spec = synth.text_spec(a.config, n=a.n)
t = synth.gen_text_device(spec, 0, spec.n)
hist = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
tot = float(hist.sum())
pats = synth.patterns(a.config, spec=spec, per_m=a.per_m, lengths=[int(x) for x in a.lengths.split(",")])
d = torch.zeros(1, dtype=torch.int64, device="cuda")

def timeit(p, strategy, peel):
    for _ in range(2):
        sm.sm_count_async(p, t, d, hist=hist, strategy=strategy, peel=peel)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        sm.sm_count_async(p, t, d, hist=hist, strategy=strategy, peel=peel)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / a.reps

for ps in pats:
    order = sm.sm_order_from_histogram(hist, ps.data)
    f = [float(hist[ps.data[j]]) / tot for j in order]
    row = {"cfg": a.config, "m": ps.m, "f": [round(x, 5) for x in f[:6]], "auto": sm.sm_plan(ps.data, hist)}
    row["filter"] = round(timeit(ps.data, 1, 0), 2)
    try:
        sm.sm_plan(ps.data, hist, strategy=3)
        for r in (1, 2, 4, 6, 8, 12):
            if r <= ps.m:
                row[f"packed{r}"] = round(timeit(ps.data, 3, r), 2)
        row["packed_auto"] = round(timeit(ps.data, 3, 0), 2)
    except sm.SmError:
        pass
    for r in (1, 2, 3, 4, 6):
        if r <= ps.m:
            row[f"block{r}"] = round(timeit(ps.data, 2, r), 2)
    print(json.dumps(row), flush=True)
