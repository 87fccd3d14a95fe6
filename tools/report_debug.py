#!/usr/bin/env python
"""Debug helper: report on small synthetic cases, print the first mismatching case (test infrastructure)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1612_01506_b200 as sm

torch.cuda.set_device(0)
rng = np.random.default_rng(1)
for n in (100, 5000, 40000, 300000, 3_000_000):
    for alpha in (b"ab", b"abcdefgh"):
        syms = np.frombuffer(alpha, dtype=np.uint8)
        a = syms[rng.integers(0, syms.size, n)]
        t = torch.from_numpy(a).cuda()
        for m in (1, 2, 5):
            p = a[:m].tobytes()
            for strat in (1, 2):
                want = oracle.naive_report(p, a)
                d = torch.zeros(1, dtype=torch.int64, device="cuda")
                pos = torch.full((want.size + 5,), -1, dtype=torch.int64, device="cuda")
                sm.sm_report_async(p, t, pos[: want.size], d, strategy=strat)
                got = pos[: want.size].cpu().numpy()
                ok = int(d.item()) == want.size and np.array_equal(got.astype(np.uint64), want)
                if not ok:
                    bad = np.nonzero(got.astype(np.uint64) != want)[0]
                    print("MISMATCH n", n, "alpha", alpha, "m", m, "strat", strat, "count", int(d.item()), want.size,
                          "first bad", bad[:5], got[bad[:5]], want[bad[:5]])
                else:
                    print("ok n", n, "alpha", alpha, "m", m, "strat", strat, "count", want.size)
