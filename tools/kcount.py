#!/usr/bin/env python
"""One batched count launch (for ncu): tools/kcount.py CONFIG M P [N_BYTES [STRATEGY]]  (sampled patterns
of length M; N_BYTES 0 = 256 MiB; STRATEGY as sm_strategy, 0 = AUTO)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1612_01506_b200 as sm
import synth
torch.cuda.set_device(0)
cfg, m, P = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
n = int(sys.argv[4]) if len(sys.argv) > 4 and int(sys.argv[4]) > 0 else (256 << 20)
strat = int(sys.argv[5]) if len(sys.argv) > 5 else 0
spec = synth.text_spec(cfg, n=n)
t = synth.gen_text_device(spec, 0, n)
h = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
pats = [p.data for p in synth.patterns(cfg, spec=spec, lengths=[m], per_m=max(P, 50)) if p.kind == "sampled"][:P]
pb = sm.PatternBatch(pats)
d = torch.zeros(pb.P, dtype=torch.int64, device="cuda")
plans = {}
for p in pats:
    s_, r_ = sm.sm_plan(p, h, strategy=strat)
    plans[(sm.STRATEGY_NAMES[s_], r_)] = plans.get((sm.STRATEGY_NAMES[s_], r_), 0) + 1
iters = int(os.environ.get("KCOUNT_ITERS", "3"))  # > 3: also the mean of the later half (sustained, power-capped)
times = []
for it in range(iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sm.sm_count_batch(pb, t, d, hist=h, strategy=strat); e1.record(); torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
ms = times[2] if iters >= 3 else times[-1]
extra = ""
if iters > 3:
    late = times[iters // 2:]
    extra = f"; sustained (iters {iters // 2}..{iters - 1}) {n * pb.P / (sum(late) / len(late)) / 1e6:.1f} GB/s"
print(f"{cfg} m={m} P={pb.P} n={n}: {ms:.3f} ms = {n * pb.P / ms / 1e6:.1f} GB/s per pattern{extra}; plans {plans}")
