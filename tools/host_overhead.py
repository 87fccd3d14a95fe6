#!/usr/bin/env python
"""Host-side enqueue time of sm_count_batch (no sync inside the loop) vs the device time, c1 sizes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1612_01506_b200 as sm
import synth
torch.cuda.set_device(0)
n = 1 << 20
spec = synth.text_spec("c1", n=n)
t = synth.gen_text_device(spec, 0, n)
h = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
pats = [p.data for p in synth.patterns("c1", spec=spec, lengths=[16], per_m=P) if p.kind == "sampled"][:P]
pb = sm.PatternBatch(pats)
d = torch.zeros(pb.P, dtype=torch.int64, device="cuda")
hd = torch.from_numpy(h.astype(np.int64)).cuda()
for label, hist in (("numpy hist", h), ("device hist", hd)):
    for _ in range(5):
        sm.sm_count_batch(pb, t, d, hist=hist)
    torch.cuda.synchronize()
    N = 200
    t0 = time.perf_counter()
    for _ in range(N):
        sm.sm_count_batch(pb, t, d, hist=hist)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"P={pb.P} {label}: host enqueue {1e6 * (t1 - t0) / N:.1f} us per call, wall per call incl. drain {1e6 * (t2 - t0) / N:.1f} us")
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    sm.sm_count_batch(pb, t, d, hist=h)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
