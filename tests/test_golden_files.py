"""The committed golden answers (tests/golden/c*.json, written by tools/make_golden.py from
oracle/ only) describe the inputs the generator makes today, and agree with the closed
forms the paper fixes where there are any.

* every pattern's SHA-256 equals that of synth.patterns(config) -- the golden counts are
  for exactly the patterns the GPU tests and bench.py use;
* c4p (t = a^(2^30)): the oracle's streamed counts equal the closed forms n - m + 1 and 0
  (PAPER.md:41-53 visits every alignment; tests/golden/closed_forms.json);
* every sampled pattern occurs (count >= 1: it was cut from the text).
"""
import hashlib
import json
import os

import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CONFIGS = ["c1", "c2", "c3", "c4", "c4p", "c5"]


def load(c):
    path = os.path.join(GOLD, f"{c}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not written yet (tools/make_golden.py {c})")
    return json.load(open(path))


@pytest.mark.parametrize("config", CONFIGS)
def test_golden_matches_generator(config):
    g = load(config)
    spec = synth.text_spec(config)
    assert g["n"] == spec.n and g["seed"] == spec.seed
    pats = synth.patterns(config, spec=spec)
    assert g["patterns"] == len(pats) == len(g["cases"])
    for c, p in zip(g["cases"], pats):
        assert (c["m"], c["start"], c["kind"]) == (p.m, p.start, p.kind)
        assert c["pattern_sha256"] == hashlib.sha256(p.data).hexdigest()
        if p.kind in ("sampled", "boundary"):
            assert c["count"] >= 1
    assert g["count_sum"] == sum(c["count"] for c in g["cases"])
    if config in ("c1", "c2"):
        assert all(len(c["positions_sha256"]) == 64 for c in g["cases"])


def test_golden_c4p_equals_closed_forms():
    g = load("c4p")
    cf = json.load(open(os.path.join(GOLD, "closed_forms.json")))
    assert g["n"] == cf["n"]
    want = {(c["m"], "b" not in c["p"]): c["count"] for c in cf["cases"]}
    for c in g["cases"]:
        assert c["count"] == want[(c["m"], c["kind"] == "periodic-match")]
