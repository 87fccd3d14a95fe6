#!/usr/bin/env python
"""Randomised parity stress (test infrastructure): random alphabets / lengths / offsets /
patterns (sampled, periodic, absent symbols), every strategy, count + report (batched and
single), against the oracle.  argv[1] = seconds (default 120)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1612_01506_b200 as sm

torch.cuda.set_device(0)
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(os.environ.get("SEED", "7")))
t_end = time.time() + secs
cases = fails = 0
while time.time() < t_end:
    sigma = int(rng.choice([1, 2, 3, 4, 5, 20, 96, 256]))
    syms = rng.choice(256, size=sigma, replace=False).astype(np.uint8)
    n = int(rng.choice([1, 2, 15, 16, 17, 100, 4095, 4096, 4097, 33000, 65536 + 7, 300001, 1 << 21]))
    skew = rng.dirichlet(np.full(sigma, 0.3 if rng.random() < 0.5 else 5.0))
    a = syms[rng.choice(sigma, size=n, p=skew)]
    if rng.random() < 0.1:
        a = np.resize(syms[rng.integers(0, sigma, int(rng.integers(1, 5)))], n)  # periodic
    off = int(rng.integers(0, 16))
    buf = torch.zeros(n + off, dtype=torch.uint8, device="cuda")
    buf[off:].copy_(torch.from_numpy(a))
    t = buf[off:]
    h = oracle.hist(a)
    pats = []
    for _ in range(int(rng.integers(1, 9))):
        m = int(rng.choice([1, 2, 2, 3, 4, 5, 8, 16, 33, 100]))
        if rng.random() < 0.7 and m <= n:
            s = int(rng.integers(0, n - m + 1))
            p = a[s:s + m].copy()
            if rng.random() < 0.2:
                p[int(rng.integers(0, m))] = syms[int(rng.integers(0, sigma))]
        else:
            p = syms[rng.integers(0, sigma, m)]
            if rng.random() < 0.2:
                p[0] = np.uint8((int(syms[0]) + 1) % 256)  # maybe absent
        pats.append(p.tobytes())
    want = [oracle.naive_count(p, a) for p in pats]
    strategies = [0, 1, 2, 4] + ([3] if sigma <= 4 else [])
    for strat in strategies:
        cases += 1
        d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        try:
            sm.sm_count_batch(pats, t, d, hist=h, strategy=strat)
        except Exception as e:  # PACKED may legitimately refuse (absent symbols)
            if strat == 3:
                continue
            raise
        if d.cpu().tolist() != want:
            fails += 1
            print("COUNT MISMATCH", sigma, n, off, strat, [len(p) for p in pats], d.cpu().tolist(), want)
            continue
        cap = sum(want)
        pos = torch.zeros(max(cap, 1), dtype=torch.int64, device="cuda")
        d2 = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        sm.sm_report_batch(pats, t, pos[:cap] if cap else None, d2, hist=h, strategy=strat)
        wp = np.concatenate([oracle.naive_report(p, a) for p in pats]) if pats else np.zeros(0)
        if d2.cpu().tolist() != want or not np.array_equal(pos[:cap].cpu().numpy().astype(np.uint64),
                                                            wp.astype(np.uint64)):
            fails += 1
            print("REPORT MISMATCH", sigma, n, off, strat, [len(p) for p in pats])
    p0 = pats[0]
    cases += 1
    if sm.sm_count(p0, t) != want[0]:
        fails += 1
        print("SINGLE COUNT MISMATCH", sigma, n, off, len(p0))
torch.cuda.synchronize()
print(f"stress parity: {cases} cases, mismatches: {fails}")
sys.exit(1 if fails else 0)
