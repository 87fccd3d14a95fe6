#!/usr/bin/env python
"""NEXT-2: executed vs algorithmic comparisons (run with SMGPU_LIB=counters on a B200).

For sampled patterns of each config stand-in (256 MiB texts; c4 = binary): the plan the
AUTO rule picks, the device counters of that launch, and the oracle's algorithmic
figures on an 8 MiB prefix:
  scalar_id   Alg. 1 character comparisons per alignment, identity order (the paper's
              "1.08 compares per alignment" statistic for English)
  scalar_freq the same with the rarest-first order (Alg. 3)
  gpu         BLOCK/PACKED: steps per warp-block (alpha_eff alignments) and executed
              compares per alignment = steps x alpha_eff / alignments;
              FILTER: queued chunk fraction, pi(1)&pi(2) survivors per alignment,
              verification compares per survivor.
Prints a markdown table."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1612_01506_b200 as sm
import synth

torch.cuda.set_device(0)
assert "counters" in sm.sm_version()
N = 256 << 20
PRE = 8 << 20
print("| config | m | plan | scalar_id | scalar_freq | gpu steps/block | gpu compares/alignment | filter queued | filter survivors/alignment | verify/survivor |")
print("|---|---|---|---|---|---|---|---|---|---|")
for cfg, lengths in (("c1", (4, 8, 16, 32)), ("c2", (2, 4, 8, 16, 64, 256)), ("c3", (4, 8, 16, 64)),
                     ("c4", (8, 32, 128))):
    spec = synth.text_spec(cfg, n=N)
    t = synth.gen_text_device(spec, 0, N)
    a = t[:PRE].cpu().numpy()
    h = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
    for m in lengths:
        pats = [p.data for p in synth.patterns(cfg, spec=spec, lengths=[m], per_m=4)][:4]
        agg = {"sid": 0.0, "sfr": 0.0, "steps": 0, "blocks": 0, "alpha": 0, "q": 0, "ch": 0, "sv": 0, "vf": 0}
        plans = set()
        for p in pats:
            s_, r_ = sm.sm_plan(p, h)
            plans.add(f"{sm.STRATEGY_NAMES[s_]}/r={r_}")
            A = PRE - m + 1
            agg["sid"] += oracle.alg4_steps(p, a, alpha=1, r=1)[0] / A
            agg["sfr"] += oracle.alg4_steps(p, a, alpha=1, pi=oracle.order(oracle.hist(a), p), r=1)[0] / A
            sm.sm_counters(reset=True)
            d = torch.zeros(1, dtype=torch.int64, device="cuda")
            sm.sm_count_async(p, t, d, hist=h)
            torch.cuda.synchronize()
            c = sm.sm_counters(reset=True)
            agg["steps"] += c["steps"]; agg["blocks"] += c["blocks"]; agg["alpha"] = max(agg["alpha"], c["alpha_eff"])
            agg["q"] += c["filter_queued"]; agg["ch"] += c["filter_chunks"]; agg["sv"] += c["filter_survivors"]
            agg["vf"] += c["filter_verify"]
        k = len(pats)
        An = (N - m + 1) * k
        blk = f"{agg['steps'] / agg['blocks']:.2f}" if agg["blocks"] else "-"
        cpa = f"{agg['steps'] * agg['alpha'] / An:.2f}" if agg["blocks"] else "-"
        q = f"{agg['q'] / agg['ch']:.4f}" if agg["ch"] else "-"
        sv = f"{agg['sv'] / An:.2e}" if agg["ch"] else "-"
        vf = f"{agg['vf'] / agg['sv']:.2f}" if agg["sv"] else "-"
        print(f"| {cfg} | {m} | {', '.join(sorted(plans))} | {agg['sid'] / k:.4f} | {agg['sfr'] / k:.4f} | {blk} | {cpa} | {q} | {sv} | {vf} |",
              flush=True)
    del t
    torch.cuda.empty_cache()
