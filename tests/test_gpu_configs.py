"""Parity at BASELINE.json's full config sizes, in the launch configuration bench.py
times (batched sm_count_batch / sm_report_batch over the device-generated text).

Every pattern of every config is compared with the oracle's golden answer
(tests/golden/c*.json, written by tools/make_golden.py from oracle/ only --
Alg. 1, and its reporting version): all counts,
and for the reporting configs c1 and c2 the SHA-256 of every pattern's
ascending position list.  Texts come from the device generator (bit-identical
to the host one the golden answers were computed on, see test_gpu_synth and
the generator digests below).  Properties that hold at any size (closed forms,
sums over all patterns, shard additivity) are checked on top.
"""
import hashlib
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sm():
    import paper_1612_01506_b200 as sm
    sm.load_library()
    return sm


def _pool():
    return ThreadPoolExecutor(max_workers=max(2, len(os.sched_getaffinity(0))))


def _free():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def golden(config):
    path = os.path.join(GOLD, f"{config}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not written (tools/make_golden.py {config})")
    g = json.load(open(path))
    spec = synth.text_spec(config)
    pats = synth.patterns(config, spec=spec)
    assert g["n"] == spec.n and len(g["cases"]) == len(pats)
    for c, p in zip(g["cases"], pats):
        assert c["pattern_sha256"] == hashlib.sha256(p.data).hexdigest()
    return g, spec, pats


def _count_all(sm, pats, t, **kw):
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch([p.data for p in pats], t, d, **kw)
    return d.cpu().numpy()


def _report_digests(sm, pats, t, total):
    """sm_report_batch over all patterns; per-pattern SHA-256 of the LE u64 positions."""
    pos = torch.empty(max(total, 1), dtype=torch.int64, device="cuda")
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_report_batch([p.data for p in pats], t, pos, d)
    cnt = d.cpu().numpy()
    host = pos[:total].cpu().numpy().astype("<u8")
    del pos
    off = np.concatenate([[0], np.cumsum(cnt)])
    assert int(off[-1]) == total
    dig = [hashlib.sha256(host[off[k]: off[k + 1]].tobytes()).hexdigest() for k in range(len(pats))]
    return cnt, dig, host, off


def test_c1_dna_all_patterns(sm):
    g, spec, pats = golden("c1")
    t = synth.gen_text_device(spec, 0, spec.n)
    a = t.cpu().numpy()
    assert np.array_equal(a, spec.host())
    want = [c["count"] for c in g["cases"]]
    assert _count_all(sm, pats, t).tolist() == want
    cnt, dig, host, off = _report_digests(sm, pats, t, sum(want))
    assert cnt.tolist() == want
    assert dig == [c["positions_sha256"] for c in g["cases"]]
    # live oracle as well (1 MiB: seconds), position by position
    with _pool() as ex:
        wpos = list(ex.map(lambda p: oracle.naive_report(p.data, a), pats))
    assert np.array_equal(host, np.concatenate(wpos))


def test_c2_english_256MiB_all_patterns(sm):
    g, spec, pats = golden("c2")
    t = synth.gen_text_device(spec, 0, spec.n)
    want = [c["count"] for c in g["cases"]]
    assert _count_all(sm, pats, t).tolist() == want            # all 1000 counts
    cnt, dig, _, _ = _report_digests(sm, pats, t, g["count_sum"])   # 142.6 M positions
    assert cnt.tolist() == want
    bad = [k for k, c in enumerate(g["cases"]) if dig[k] != c["positions_sha256"]]
    assert not bad, f"{len(bad)} position lists differ, first pattern {bad[:5]}"
    del t
    _free()


def test_c3_protein_1GiB_all_patterns(sm):
    g, spec, pats = golden("c3")
    assert len(pats) == 7 * 120
    t = synth.gen_text_device(spec, 0, spec.n)
    assert _count_all(sm, pats, t).tolist() == [c["count"] for c in g["cases"]]
    del t
    _free()


def test_c4_binary_4GiB_all_patterns(sm):
    g, spec, pats = golden("c4")
    t = synth.gen_text_device(spec, 0, spec.n)
    n = spec.n
    assert _count_all(sm, pats, t).tolist() == [c["count"] for c in g["cases"]]
    # sum over ALL 2^k patterns of length k over {0,1} = n - k + 1 (every alignment matches one)
    for k in (1, 8):
        allp = [bytes((v >> (k - 1 - j)) & 1 for j in range(k)) for v in range(1 << k)]
        d = torch.zeros(len(allp), dtype=torch.int64, device="cuda")
        sm.sm_count_batch(allp, t, d)
        assert int(d.sum().item()) == n - k + 1
    h = sm.sm_histogram(t).cpu().numpy()
    assert int(h[0]) + int(h[1]) == n
    del t
    _free()


def test_c4_periodic_closed_forms(sm):
    g, spec, pats = golden("c4p")
    t = synth.gen_text_device(spec, 0, spec.n)
    assert _count_all(sm, pats, t).tolist() == [c["count"] for c in g["cases"]]
    cf = json.load(open(os.path.join(GOLD, "closed_forms.json")))
    assert spec.n == cf["n"]
    cpats = [b"a" * c["m"] if c["p"].startswith("a^") and "b" not in c["p"] else b"a" * (c["m"] - 1) + b"b"
             for c in cf["cases"]]
    d = torch.zeros(len(cpats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch(cpats, t, d)
    assert d.cpu().tolist() == [c["count"] for c in cf["cases"]]
    # NEXT-1 dense reporting: p = a^17 occurs at every alignment 0 .. n - 17 (2^30 - 16
    # positions, 8 GiB of output); positions are unique, so compare them all, in slices
    m = 17
    want = spec.n - m + 1
    pos = torch.empty(want, dtype=torch.int64, device="cuda")
    d1 = torch.zeros(1, dtype=torch.int64, device="cuda")
    sm.sm_report_batch([b"a" * m], t, pos, d1)
    assert int(d1.item()) == want
    step = 1 << 27
    for lo in range(0, want, step):
        hi = min(want, lo + step)
        assert torch.equal(pos[lo:hi], torch.arange(lo, hi, dtype=torch.int64, device="cuda")), lo
    del pos, t
    _free()


def test_c5_uniform_64GiB_all_patterns(sm):
    from paper_1612_01506_b200 import dist
    spec = synth.text_spec("c5")
    N = spec.n
    free, _ = torch.cuda.mem_get_info()
    if free < N + (4 << 30):
        pytest.skip("needs 68 GiB of free device memory")
    g, spec, pats = golden("c5")
    assert len(pats) == 200
    t = synth.gen_text_device(spec, 0, N)
    data = [p.data for p in pats]
    full = _count_all(sm, pats, t)
    assert full.tolist() == [c["count"] for c in g["cases"]]   # incl. 28 boundary patterns per m
    # shard additivity: G = 2, 4, 8 ranks' owned counts sum to the oracle's count
    h = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
    for G in (2, 4, 8):
        tot = np.zeros(len(pats), dtype=np.int64)
        for sh in dist.all_shards(N, G, halo=63):
            c = dist.count_sharded(data, t[sh.own_lo: sh.held_hi], sh, hist=h)
            tot += c.cpu().numpy()
        assert np.array_equal(tot, full), G
    del t
    _free()
