#!/usr/bin/env python
"""Kernel microbenchmark: per-launch time of the count kernel, per pattern length.

Times R back-to-back batches of sm_count_async launches with two CUDA events
(no per-launch events), so the number is the average launch duration including
inter-launch gaps.  Knobs come from SMGPU_* env variables (see abi.cu Tunables).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1612_01506_b200 as sm
import synth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--lengths", default="2,8,64,1024")
    ap.add_argument("--per-m", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--strategy", type=int, default=0)
    ap.add_argument("--peel", type=int, default=0)
    ap.add_argument("--tag", default="")
    ap.add_argument("--batch", action="store_true", help="time sm_count_batch over the m's patterns")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    spec = synth.text_spec(a.config, n=a.n)
    t = synth.gen_text_device(spec, 0, spec.n)
    hist = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
    lengths = [int(x) for x in a.lengths.split(",")]
    pats = synth.patterns(a.config, spec=spec, per_m=a.per_m, lengths=lengths)
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    res = {"tag": a.tag, "config": spec.name, "n": spec.n,
           "env": {k: v for k, v in os.environ.items() if k.startswith("SMGPU_")}}
    for m in lengths:
        ps = [p for p in pats if p.m == m]
        if a.batch:
            pb = sm.PatternBatch([p.data for p in ps])
            for _ in range(2):
                sm.sm_count_batch(pb, t, d, hist=hist, strategy=a.strategy)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                sm.sm_count_batch(pb, t, d, hist=hist, strategy=a.strategy)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (a.reps * len(ps))
            res[str(m)] = {"us": round(us, 2), "GBps": round(spec.n / us / 1e3, 1), "host_us": 0}
            continue
        for _ in range(2):
            for i, p in enumerate(ps):
                sm.sm_count_async(p.data, t, d[i:i + 1], hist=hist, strategy=a.strategy, peel=a.peel)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            for i, p in enumerate(ps):
                sm.sm_count_async(p.data, t, d[i:i + 1], hist=hist, strategy=a.strategy, peel=a.peel)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (a.reps * len(ps))
        # host enqueue cost per call (GPU kept busy by a long first batch)
        import time
        h0 = time.perf_counter()
        for i, p in enumerate(ps):
            sm.sm_count_async(p.data, t, d[i:i + 1], hist=hist, strategy=a.strategy, peel=a.peel)
        host_us = (time.perf_counter() - h0) * 1e6 / len(ps)
        torch.cuda.synchronize()
        plans = {}
        for p in ps:
            s, r = sm.sm_plan(p.data, hist, strategy=a.strategy, peel=a.peel)
            plans[f"{s}/{r}"] = plans.get(f"{s}/{r}", 0) + 1
        res[str(m)] = {"us": round(us, 2), "GBps": round(spec.n / us / 1e3, 1), "host_us": round(host_us, 1), "plans": plans}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
