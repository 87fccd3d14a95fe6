"""Write oracle golden answers for every pattern of the five BASELINE.json configs.

    python tools/make_golden.py [c1 c2 c3 c4 c4p c5] [--threads N]

Calls ONLY ``oracle/`` (Alg. 1 Naive-search, and its reporting
version) on texts and patterns from ``synth/`` (the seeded input
generator, no method arithmetic).  Nothing here touches the CUDA path.

Output: ``tests/golden/<config>.json`` with, per pattern (in ``synth.patterns``
order): m, start, kind, SHA-256 of the pattern bytes, the occurrence count, and
for the reporting configs (c1, c2) the SHA-256 of the ascending 0-based
positions as little-endian u64.

Large texts are streamed: the text is generated in blocks of ``BLOCK`` bytes
(deliberately NOT a power of two, so block cuts never coincide with the C5 shard
cuts a_k = k*N/8 nor with the GPU's 32 KiB tiles) plus an (m_max-1)-byte overlap,
and the oracle counts, for each pattern, the alignments i of the block
[lo, hi) by running Alg. 1 on t[lo .. min(hi + m - 1, n)) -- the count of a
text slice is the definition restricted to that slice.  Per-block counts are
summed; position lists are hashed block after block, which keeps them in
ascending order.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
BLOCK = (1 << 28) + 4099 * 16 + 5          # odd-sized blocks: cuts unaligned to shards/tiles
REPORT = {"c1", "c2"}                       # configs whose positions are recorded (BASELINE.json)


def golden(config: str, threads: int, n: int | None = None, per_m: int | None = None,
           block: int = BLOCK) -> dict:
    """Golden answers of `config` (n / per_m override the sizes: tests of the streaming only)."""
    spec = synth.text_spec(config, n=n)
    n = spec.n
    t0 = time.time()
    pats = synth.patterns(config, spec=spec, per_m=per_m)
    P = len(pats)
    mmax = max(p.m for p in pats)
    report = config in REPORT
    counts = [0] * P
    hashers = [hashlib.sha256() for _ in range(P)] if report else None
    nblocks = (n + block - 1) // block
    # sub-range splitting so that few-pattern configs (c4p) still use every thread
    splits = max(1, -(-2 * threads // P))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        nxt = ex.submit(spec.host, 0, min(n, block + mmax - 1))
        for b in range(nblocks):
            lo = b * block
            hi = min(n, lo + block)
            text = nxt.result()
            if b + 1 < nblocks:
                lo2 = hi
                nxt = ex.submit(spec.host, lo2, min(n, lo2 + block + mmax - 1) - lo2)

            def work(item):
                k, a, z = item               # alignments [a, z) of pattern k, block-relative
                m = pats[k].m
                seg = text[a: min(z + m - 1, text.size)]
                if report:
                    return k, oracle.naive_report(pats[k].data, seg) + np.uint64(lo + a)
                return k, oracle.naive_count(pats[k].data, seg)

            items = []
            for k, p in enumerate(pats):
                last = min(hi, n - p.m + 1) - lo     # alignments of this block: [0, last)
                if last <= 0:
                    continue
                step = -(-last // splits)
                for s in range(splits):
                    a, z = s * step, min(last, (s + 1) * step)
                    if a < z:
                        items.append((k, a, z))
            # ex.map preserves item order, so each pattern's sub-ranges hash in ascending order
            for k, res in ex.map(work, items):
                if report:
                    counts[k] += int(res.size)
                    hashers[k].update(np.ascontiguousarray(res, dtype="<u8").tobytes())
                else:
                    counts[k] += int(res)
            if nblocks > 1:
                print(f"  {config}: block {b + 1}/{nblocks} done, {time.time() - t0:.0f} s", flush=True)
    out = []
    for k, p in enumerate(pats):
        e = {"m": p.m, "start": p.start, "kind": p.kind,
             "pattern_sha256": hashlib.sha256(p.data).hexdigest(), "count": counts[k]}
        if report:
            e["positions_sha256"] = hashers[k].hexdigest()
        out.append(e)
    return {
        "config": config,
        "text": spec.name,
        "n": n,
        "seed": spec.seed,
        "source": ("oracle.naive_count / oracle.naive_report (Alg. 1, PAPER.md:41-53; reporting "
                   "PAPER.md:36) over synth-generated text, streamed in blocks of "
                   f"{block} B with an (m-1)-byte overlap; written by tools/make_golden.py"),
        "positions": "sha256 of ascending 0-based positions, little-endian u64" if report else None,
        "patterns": len(out),
        "count_sum": int(sum(counts)),
        "oracle_seconds": round(time.time() - t0, 1),
        "threads": threads,
        "cases": out,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1", "c2", "c3", "c4", "c4p", "c5"])
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    a = ap.parse_args()
    os.makedirs(GOLD, exist_ok=True)
    for c in a.configs:
        g = golden(c, a.threads)
        path = os.path.join(GOLD, f"{c}.json")
        with open(path + ".tmp", "w") as f:
            json.dump(g, f, indent=0)
        os.replace(path + ".tmp", path)
        print(f"{c}: {g['patterns']} patterns, count_sum {g['count_sum']}, {g['oracle_seconds']} s -> {path}",
              flush=True)


if __name__ == "__main__":
    main()
