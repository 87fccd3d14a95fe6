#!/usr/bin/env python
"""Dense case a^(2^30), p = a^m: count vs report timing (with the histogram given), per strategy."""
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
hist = sm.sm_histogram(t).cpu().numpy().astype("uint64")
pos = torch.empty(total, dtype=torch.int64, device="cuda")
d = torch.zeros(1, dtype=torch.int64, device="cuda")
pb = sm.PatternBatch([b"a" * m])
def timeit(f, reps=3):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
for name, strat in (("auto", sm.SM_STRATEGY_AUTO), ("filter", sm.SM_STRATEGY_FILTER), ("block", sm.SM_STRATEGY_BLOCK),
                    ("packed", sm.SM_STRATEGY_PACKED)):
    try:
        c = timeit(lambda: sm.sm_count_batch(pb, t, d, hist=hist, strategy=strat))
        assert int(d.item()) == total
        r = timeit(lambda: sm.sm_report_batch(pb, t, pos, d, hist=hist, strategy=strat))
        assert int(d.item()) == total and int(pos[-1].item()) == total - 1
        print(f"{name:7s} count {c:.3f} ms  report {r:.3f} ms  ({(spec.n + 8 * total) / r / 1e6:.0f} GB/s r+w)")
    except Exception as e:  # noqa: BLE001
        print(name, "error", e)
