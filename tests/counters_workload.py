#!/usr/bin/env python
"""NEXT-2 compare-step counters (run with SMGPU_LIB=counters by tests/test_gpu_counters.py).

The instrumented library counts, per launch, the SIMDcompare steps the BLOCK / PACKED
kernels execute over their warp-blocks of 512 x CPL consecutive alignments (Alg. 4,
PAPER.md:151-174, at alpha = the warp's span) and the survivors of FILTER's two peeled
comparisons.  Pinned here against the oracle (test infrastructure): the step count must
equal oracle.alg4_steps(p, t, alpha_eff, pi, r) exactly -- i.e. the kernel executes
Alg. 4's early exits, no more and no fewer compares -- and FILTER's survivors must equal
the number of valid alignments matching pi(1) and pi(2), counted with numpy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1612_01506_b200 as sm

torch.cuda.set_device(0)
assert "counters" in sm.sm_version(), sm.sm_version()
rng = np.random.default_rng(77)
fails = 0


def run(p, a, t, strategy, order=None, peel=0):
    sm.sm_counters(reset=True)
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    h = oracle.hist(a)
    sm.sm_count_async(p, t, d, hist=h, order=order, peel=peel, strategy=strategy)
    got = int(d.item())
    return got, sm.sm_counters(reset=True)


cases = []
for n in ((1 << 20) + 333, (16 << 20) + 77):
    for alpha_syms in (b"a", b"ACGT", b"\x00\x01", bytes(range(97, 123))):
        syms = np.frombuffer(alpha_syms, dtype=np.uint8)
        a = syms[rng.integers(0, syms.size, n)]
        t = torch.from_numpy(a).cuda()        # a fresh allocation: 16-B aligned (delta = 0)
        for m in (1, 3, 8, 21):
            s0 = int(rng.integers(0, n - m + 1))
            p = a[s0:s0 + m].tobytes()
            h = oracle.hist(a)
            pi = oracle.order(h, p)
            for strategy in (sm.SM_STRATEGY_BLOCK, sm.SM_STRATEGY_PACKED):
                if strategy == sm.SM_STRATEGY_PACKED and syms.size > 4:
                    continue
                for peel in (1, 2, 5):
                    got, c = run(p, a, t, strategy, order=pi.tolist(), peel=peel)
                    want = oracle.naive_count(p, a)
                    steps, blocks = oracle.alg4_steps(p, a, alpha=c["alpha_eff"], pi=pi, r=peel)
                    ok = got == want and c["steps"] == steps and c["blocks"] == blocks
                    fails += not ok
                    print(("ok " if ok else "MISMATCH ") + f"n={n} sigma={syms.size} m={m} strat={strategy} r={peel} "
                          f"alpha={c['alpha_eff']} steps={c['steps']}/{steps} blocks={c['blocks']}/{blocks} "
                          f"count={got}/{want}")
            if syms.size <= 4:  # batches of >= 2 patterns run PACKED on the text's code array (NEXT-3)
                sm.sm_counters(reset=True)
                d2 = torch.zeros(2, dtype=torch.int64, device="cuda")
                sm.sm_count_batch([p, p], t, d2, hist=oracle.hist(a), strategy=sm.SM_STRATEGY_PACKED)
                c = sm.sm_counters(reset=True)
                pi_auto = oracle.order(oracle.hist(a), p)
                r_auto = sm.sm_plan(p, oracle.hist(a), strategy=sm.SM_STRATEGY_PACKED)[1]
                steps, blocks = oracle.alg4_steps(p, a, alpha=c["alpha_eff"], pi=pi_auto, r=r_auto)
                want = oracle.naive_count(p, a)
                ok = d2.cpu().tolist() == [want, want] and c["steps"] == 2 * steps and c["blocks"] == 2 * blocks
                fails += not ok
                print(("ok " if ok else "MISMATCH ") + f"PRE-PACKED batch n={n} sigma={syms.size} m={m} "
                      f"steps={c['steps']}/{2 * steps} blocks={c['blocks']}/{2 * blocks}")
            for fs in (sm.SM_STRATEGY_FILTER, sm.SM_STRATEGY_PAIR):  # survivors of pi(1), pi(2)
                if m < 2:
                    break
                got, c = run(p, a, t, fs, order=pi.tolist())
                A = n - m + 1
                a1, a2 = int(pi[0]), int(pi[1])
                surv = int(np.count_nonzero((a[a1:a1 + A] == p[a1]) & (a[a2:a2 + A] == p[a2])))
                ok = c["filter_survivors"] == surv and got == oracle.naive_count(p, a)
                fails += not ok
                print(("ok " if ok else "MISMATCH ") + f"FILTER/PAIR({fs}) n={n} sigma={syms.size} m={m} "
                      f"survivors={c['filter_survivors']}/{surv} queued={c['filter_queued']} verify={c['filter_verify']}")
print("counters workload done, mismatches:", fails)
sys.exit(1 if fails else 0)
