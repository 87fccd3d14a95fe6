#!/usr/bin/env python
"""One count batch and one report batch over the same c2 patterns (for ncu comparison of the
kEpiCount and kEpiStage search kernels).  argv[1] = pattern length (default 16), argv[2] = patterns."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1612_01506_b200 as sm
import synth
torch.cuda.set_device(0)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
P = int(sys.argv[2]) if len(sys.argv) > 2 else 64
spec = synth.text_spec("c2")
t = synth.gen_text_device(spec, 0, spec.n)
hist = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
pats = sm.PatternBatch([p.data for p in synth.patterns("c2", spec=spec, lengths=[m], per_m=P)])
d = torch.zeros(pats.P, dtype=torch.int64, device="cuda")
sm.sm_count_batch(pats, t, d, hist=hist)
tot = int(d.sum().item())
pos = torch.empty(max(tot, 1), dtype=torch.int64, device="cuda")
d2 = torch.zeros(pats.P, dtype=torch.int64, device="cuda")
sm.sm_report_batch(pats, t, pos, d2, hist=hist)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
ev[0].record(); sm.sm_count_batch(pats, t, d, hist=hist); ev[1].record()
sm.sm_report_batch(pats, t, pos, d2, hist=hist); ev[2].record(); torch.cuda.synchronize()
print(f"m={m} P={pats.P} count {ev[0].elapsed_time(ev[1]):.3f} ms  report {ev[1].elapsed_time(ev[2]):.3f} ms  positions {tot}")
