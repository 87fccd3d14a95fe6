#!/usr/bin/env python
"""Edge-case workload for the bounds-checked build (tests/test_gpu_debug_checks.py): every strategy x epilogue, unaligned views,
ragged ends, batches; checks results against the oracle (test infrastructure)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1612_01506_b200 as sm

torch.cuda.set_device(0)
print("library:", sm.load_library()._name, "SMGPU_STAGE_BYTES:", os.environ.get("SMGPU_STAGE_BYTES"))
rng = np.random.default_rng(2024)
fails = 0
SMALL = os.environ.get("SMGPU_WORKLOAD_SMALL") == "1"  # compute-sanitizer runs (tools/sanitize.sh)
for alpha in (b"ACGT", b"\x00\x01", bytes(range(32, 127)), b"a"):
    syms = np.frombuffer(alpha, dtype=np.uint8)
    for n in ((5, 31, 4100) if SMALL else (5, 31, 4100, 70003)):
        a = syms[rng.integers(0, syms.size, n)]
        h = oracle.hist(a)
        for off in (0, 3, 15):
            buf = torch.zeros(n + off, dtype=torch.uint8, device="cuda")
            buf[off:].copy_(torch.from_numpy(a))
            t = buf[off:]                          # the allocation ends exactly at t + n
            pats = []
            for m in (1, 2, 3, 17, 40):
                if m <= n:
                    s = int(rng.integers(0, n - m + 1))
                    pats.append(a[s:s + m].tobytes())
            strategies = [1, 2, 4] + ([3] if len(alpha) <= 4 else [])
            for strat in strategies:
                d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
                sm.sm_count_batch(pats, t, d, hist=h, strategy=strat)
                want = [oracle.naive_count(p, a) for p in pats]
                fails += d.cpu().tolist() != want
                cap = sum(want)
                pos = torch.zeros(max(cap, 1), dtype=torch.int64, device="cuda")
                d2 = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
                sm.sm_report_batch(pats, t, pos[:cap] if cap else None, d2, hist=h, strategy=strat)
                wp = np.concatenate([oracle.naive_report(p, a) for p in pats]) if pats else np.zeros(0)
                fails += not np.array_equal(pos[:cap].cpu().numpy().astype(np.uint64), wp.astype(np.uint64))
            fails += sm.sm_histogram(t).cpu().numpy().astype(np.uint64).tolist() != h.tolist()
            for p in pats[:2]:  # the single-pattern entry points (their own launch path)
                fails += sm.sm_count(p, t) != oracle.naive_count(p, a)
                got, tot = sm.sm_report(p, t)
                fails += tot != oracle.naive_count(p, a) or not np.array_equal(
                    got.cpu().numpy().astype(np.uint64), oracle.naive_report(p, a).astype(np.uint64))
# dense reports that fill the staging pool (every alignment matches): with a small
# SMGPU_STAGE_BYTES the tiles split between staged records and the overflow pass
for n in ((70003,) if SMALL else (70003, 300001)):
    a = np.full(n, ord("a"), dtype=np.uint8)
    t = torch.from_numpy(a).cuda()
    pats = [b"a", b"aa", b"a" * 17]
    want = [n - len(p) + 1 for p in pats]
    for cap in (sum(want), 10, 4000):
        pos = torch.zeros(cap, dtype=torch.int64, device="cuda")
        d2 = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        sm.sm_report_batch(pats, t, pos, d2)
        fails += d2.cpu().tolist() != want
        wp = np.concatenate([np.arange(w, dtype=np.uint64) for w in want])[:cap]
        fails += not np.array_equal(pos.cpu().numpy().astype(np.uint64), wp)
# an advisory (wrong) caller histogram: ACGT-only for a text with 'N' bytes
a = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, 9000)].copy()
a[::97] = ord("N")
h = np.zeros(256, dtype=np.uint64)
h[list(b"ACGT")] = 1
t = torch.from_numpy(a).cuda()
pats = [b"G", b"GN", b"AGG", a[50:70].tobytes()]
for strat in (0, 3):
    sel = [p for p in pats if strat == 0 or b"N" not in p]
    d = torch.zeros(len(sel), dtype=torch.int64, device="cuda")
    sm.sm_count_batch(sel, t, d, hist=h, strategy=strat)
    fails += d.cpu().tolist() != [oracle.naive_count(p, a) for p in sel]
torch.cuda.synchronize()
print("sanitize workload done, mismatches:", fails)
sys.exit(1 if fails else 0)
