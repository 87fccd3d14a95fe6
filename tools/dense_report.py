#!/usr/bin/env python
"""NEXT-1 dense reporting: a^(2^30) with p = a^17 (every alignment matches, 8 GiB of positions);
prints ms and read+write GB/s (for an ncu launch list of the reporting kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_01506_b200 as sm
import synth
torch.cuda.set_device(0)
spec = synth.text_spec("c4p")
t = synth.gen_text_device(spec, 0, spec.n)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 17
total = spec.n - m + 1
pos = torch.empty(total, dtype=torch.int64, device="cuda")
d = torch.zeros(1, dtype=torch.int64, device="cuda")
pb = sm.PatternBatch([b"a" * m])
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sm.sm_report_batch(pb, t, pos, d); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"dense report m={m}: {ms:.3f} ms, {(spec.n + 8 * total) / ms / 1e6:.1f} GB/s read+write, count {int(d.item())}")
assert int(d.item()) == total and int(pos[-1].item()) == total - 1
