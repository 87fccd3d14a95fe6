#!/usr/bin/env python
"""One bench step's batched count launches over the c2 workload (for `ncu --set full` of a
single search_kernel launch, e.g. -k regex:search_kernel --launch-skip 4 -c 1).
Prints each launch's pattern count so the capture can be converted to per-pattern figures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1612_01506_b200 as sm
import synth
torch.cuda.set_device(0)
spec = synth.text_spec("c2")
t = synth.gen_text_device(spec, 0, spec.n)
h = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
pats = [p.data for p in synth.patterns("c2", spec=spec)]
pb = sm.PatternBatch(pats)
d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
sm.sm_count_batch(pb, t, d, hist=h)
torch.cuda.synchronize()
# the launch grouping of sm_count_batch: per strategy, <= 64 patterns and <= 6400 table words
groups = {}
for p in pats:
    s_, _ = sm.sm_plan(p, h)
    groups.setdefault(s_, []).append(len(p))
launches = []
for s_, ms in groups.items():
    cur, words = 0, 0
    for m in ms:
        if cur == 64 or words + m > 6400:
            launches.append((s_, cur))
            cur, words = 0, 0
        cur += 1
        words += m
    if cur:
        launches.append((s_, cur))
print("launches (strategy, patterns) in issue order is by first-full batch; groups:",
      {sm.STRATEGY_NAMES[k]: len(v) for k, v in groups.items()})
print("batches:", launches)
