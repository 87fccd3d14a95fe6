"""The golden-answer writer's streaming (tools/make_golden.py) equals one whole-text oracle call.

Blocks of a few KiB (odd sizes, so cuts fall inside occurrences) with the
(m-1)-byte overlap must give exactly the counts and position digests of
Alg. 1 (reporting PAPER.md:36) run once over the whole text.
"""
import hashlib
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import oracle  # noqa: E402
import synth  # noqa: E402
import make_golden  # noqa: E402


@pytest.mark.parametrize("config,n,block", [("c1", 50_000, 4099), ("c2", 70_001, 5003),
                                             ("c4", 40_000, 3001), ("c4p", 3000, 1001),
                                             ("c5", 1 << 16, 7777), ("c3", 30_000, 9999)])
def test_streamed_equals_whole(config, n, block):
    g = make_golden.golden(config, threads=3, n=n, per_m=3, block=block)
    spec = synth.text_spec(config, n=n)
    t = spec.host()
    pats = synth.patterns(config, spec=spec, per_m=3)
    assert g["patterns"] == len(pats)
    for c, p in zip(g["cases"], pats):
        assert c["pattern_sha256"] == hashlib.sha256(p.data).hexdigest()
        assert c["count"] == oracle.naive_count(p.data, t), (p.m, p.kind)
        if "positions_sha256" in c:
            pos = oracle.naive_report(p.data, t).astype("<u8")
            assert c["positions_sha256"] == hashlib.sha256(pos.tobytes()).hexdigest()
    assert g["count_sum"] == sum(c["count"] for c in g["cases"])


def test_c5_boundary_patterns_span_block_cuts():
    """c5's boundary patterns straddle the 8-way shard cuts; the writer's block size is
    chosen so its own cuts are different ones (each cut is tested by one of the two)."""
    N = 1 << 36
    cuts = set(synth.c5_boundaries(N))
    assert not any(b * make_golden.BLOCK in cuts for b in range(1, N // make_golden.BLOCK + 1))
    assert make_golden.BLOCK % 16 != 0
