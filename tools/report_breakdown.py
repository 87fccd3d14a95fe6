#!/usr/bin/env python
"""One sm_report_batch call over the c2 pattern set (for an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1612_01506_b200 as sm
import synth
torch.cuda.set_device(0)
spec = synth.text_spec("c2")
t = synth.gen_text_device(spec, 0, spec.n)
hist = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
lengths = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else None
pats = sm.PatternBatch([p.data for p in synth.patterns("c2", spec=spec, lengths=lengths)])
d = torch.zeros(pats.P, dtype=torch.int64, device="cuda")
sm.sm_count_batch(pats, t, d, hist=hist)
tot = int(d.sum().item())
pos = torch.empty(max(tot, 1), dtype=torch.int64, device="cuda")
d2 = torch.zeros(pats.P, dtype=torch.int64, device="cuda")
for _ in range(2):
    sm.sm_report_batch(pats, t, pos, d2, hist=hist)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); sm.sm_report_batch(pats, t, pos, d2, hist=hist); e1.record(); torch.cuda.synchronize()
print("report ms", e0.elapsed_time(e1), "positions", tot, "patterns", pats.P)
