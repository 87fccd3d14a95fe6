#!/usr/bin/env python
"""NEXT-2 refreshed on the round-2 build: order ablation and r sweep, batched.

* Orders (PAPER.md:184-186 fixed orders vs the frequency order of PAPER.md:113,138 --
  the N32 / N32-fixed / N32-freq columns of Tables 1-4): identity, pi_h, pi_hs, freq, for
  BLOCK (the paper's Alg. 4, r = 2 for freq / 3 otherwise), FILTER and AUTO.
* r sweep (r = 2 English, r = 3 theory / 5 practice for DNA, r = 3 for
  large alphabets): r = 1..8 for BLOCK / PACKED (the strategies that peel)
  against AUTO, on c1-like DNA, c3 protein and c4 binary texts.

Every variant is one sm_count_batch_ordered call over the same patterns (the bench's
launch configuration: 3 CTAs per SM, counter dispatch), timed with CUDA events,
best of --reps; counts are checked equal across variants (orders and r never change them).
Output: one JSON line per (config, m), text GB/s per variant."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1612_01506_b200 as sm
import synth


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", choices=["orders", "rsweep"], default="orders")
    ap.add_argument("--configs", default="c2,c3,c1")
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--lengths", default="4,8,16,32,64")
    ap.add_argument("--per-m", type=int, default=16)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rmax", type=int, default=8)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for cfg in a.configs.split(","):
        spec = synth.text_spec(cfg, n=a.n)
        t = synth.gen_text_device(spec, 0, spec.n)
        hist = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
        lengths = [int(x) for x in a.lengths.split(",")]
        pats = synth.patterns(cfg, spec=spec, per_m=a.per_m, lengths=lengths)
        for m in lengths:
            ps = [p.data for p in pats if p.m == m and p.kind == "sampled"]
            pb = sm.PatternBatch(ps)
            d = torch.zeros(len(ps), dtype=torch.int64, device="cuda")
            row = {"cfg": cfg, "n": spec.n, "m": m, "patterns": len(ps)}
            ref = None
            variants = []
            if a.mode == "orders":
                for oname in ("identity", "pi_h", "pi_hs", "freq"):
                    orders = None if oname == "freq" else [
                        sm.sm_heuristic_order(p, {"identity": 0, "pi_h": 1, "pi_hs": 2}[oname]) for p in ps]
                    for sname, strat, peel in (("block", sm.SM_STRATEGY_BLOCK, 2 if oname == "freq" else 3),
                                               ("filter", sm.SM_STRATEGY_FILTER, 0), ("auto", 0, 0)):
                        variants.append((f"{sname}/{oname}", orders, [peel] * len(ps), strat))
            else:
                packed = int((hist > 0).sum()) <= 4
                strat = sm.SM_STRATEGY_PACKED if packed else sm.SM_STRATEGY_BLOCK
                sname = "packed" if packed else "block"
                variants.append(("auto", None, None, 0))
                for r in range(1, a.rmax + 1):
                    variants.append((f"{sname}/r={r}", None, [r] * len(ps), strat))
                row["auto_plan"] = [sm.STRATEGY_NAMES[x] + f"/r={y}" for x, y in [sm.sm_plan(ps[0], hist)]]
            for name, orders, peels, strat in variants:
                ms = timed(lambda: sm.sm_count_batch_ordered(pb, t, d, orders=orders, peels=peels, hist=hist,
                                                             strategy=strat), a.reps)
                got = d.cpu().tolist()
                if ref is None:
                    ref = got
                assert got == ref, (cfg, m, name)
                row[name] = round(spec.n * len(ps) / (ms * 1e-3) / 1e9, 1)
            print(json.dumps(row), flush=True)
        del t
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
