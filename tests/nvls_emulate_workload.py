#!/usr/bin/env python
"""NEXT-4 last-CTA epilogue protocol on one GPU (run with SMGPU_NVLS_EMULATE=1 by
tests/test_gpu_nvls.py): sm_count_batch_multicast with a plain device buffer as
mc_counts, the epilogue's multimem.red replaced by an atomic add.  Checks, against the
oracle, that every pattern's count arrives exactly once per call (all CTAs' atomics are
in before the last CTA reads them; no launch adds twice) -- over batches that need
several launches, guarded PACKED launches with their fallbacks, and shard limits."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1612_01506_b200 as sm
import synth

torch.cuda.set_device(0)
fails = 0
cases = [("c2", (8 << 20) + 77, 12), ("c1", (4 << 20) + 3, 40), ("c3", (16 << 20) + 5, 20)]
for cfg, n, per_m in cases:
    spec = synth.text_spec(cfg, n=n)
    t = synth.gen_text_device(spec, 0, spec.n)
    a = t.cpu().numpy()
    pats = [p.data for p in synth.patterns(cfg, spec=spec, per_m=per_m)]   # > 64: several launches
    h = oracle.hist(a)
    for hist, lim in ((h, None), (None, spec.n // 3), (h, spec.n // 2)):
        mc = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        for rep in range(2):  # accumulates: two calls add twice
            sm.sm_count_batch_multicast(pats, t, mc.data_ptr(), hist=hist, max_alignments=lim)
        torch.cuda.synchronize()
        L = spec.n if lim is None else lim
        want = np.array([2 * oracle.naive_count(p, a[: min(spec.n, L + len(p) - 1)]) for p in pats])
        ok = np.array_equal(mc.cpu().numpy(), want)
        fails += not ok
        print(("ok " if ok else "MISMATCH ") + f"{cfg} n={n} P={len(pats)} lim={lim} hist={'caller' if hist is not None else 'device'}")
print("nvls emulate workload done, mismatches:", fails)
sys.exit(1 if fails else 0)
