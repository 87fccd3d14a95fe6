"""Parity at BASELINE.json's full config sizes, in the launch configuration bench.py
times (batched sm_count_batch / sm_report_batch over the device-generated text).

Texts come from the device generator (bit-identical to the host one, see
test_gpu_synth) and are copied back to the host for the oracle.  Where the
oracle can afford it, sampled outputs are compared element by element (oracle
calls run in parallel threads; ctypes releases the GIL); at 4 GiB and 64 GiB
the checks are properties that hold at any size (closed forms, sums over all
patterns, shard additivity, sampled patterns occur).
"""
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


def test_c1_dna_all_patterns(sm):
    spec = synth.text_spec("c1")
    t = synth.gen_text_device(spec, 0, spec.n)
    a = t.cpu().numpy()
    assert np.array_equal(a, spec.host())
    pats = [p.data for p in synth.patterns("c1", spec=spec)]
    assert len(pats) == 200
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch(pats, t, d)
    with _pool() as ex:
        want = list(ex.map(lambda p: oracle.naive_count(p, a), pats))
    assert d.cpu().tolist() == want
    tot = int(sum(want))
    pos = torch.zeros(tot, dtype=torch.int64, device="cuda")
    d2 = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_report_batch(pats, t, pos, d2)
    with _pool() as ex:
        wpos = list(ex.map(lambda p: oracle.naive_report(p, a), pats))
    assert d2.cpu().tolist() == want
    assert np.array_equal(pos.cpu().numpy().astype(np.uint64), np.concatenate(wpos))


def test_c2_english_256MiB(sm):
    spec = synth.text_spec("c2")
    t = synth.gen_text_device(spec, 0, spec.n)
    a = t.cpu().numpy()
    pats = synth.patterns("c2", spec=spec)  # 1000 patterns, the bench workload
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch([p.data for p in pats], t, d)
    got = d.cpu().numpy()
    assert (got >= 1).all()  # every pattern was sampled from the text
    # element-wise oracle parity on 2 sampled patterns per length (20 full-text scans)
    idx = [i for m in synth.PATTERN_LENGTHS["c2"] for i in [j for j, p in enumerate(pats) if p.m == m][:2]]
    with _pool() as ex:
        want = list(ex.map(lambda i: oracle.naive_count(pats[i].data, a), idx))
    assert [int(got[i]) for i in idx] == want
    # reporting: the densest m = 2 pattern and two m = 8 patterns, position by position
    sel = [max((i for i, p in enumerate(pats) if p.m == 2), key=lambda i: got[i])] + \
          [i for i, p in enumerate(pats) if p.m == 8][:2]
    sub = [pats[i].data for i in sel]
    cap = int(sum(got[i] for i in sel))
    pos = torch.zeros(cap, dtype=torch.int64, device="cuda")
    d2 = torch.zeros(len(sel), dtype=torch.int64, device="cuda")
    sm.sm_report_batch(sub, t, pos, d2)
    with _pool() as ex:
        wpos = list(ex.map(lambda p: oracle.naive_report(p, a), sub))
    assert d2.cpu().tolist() == [w.size for w in wpos]
    assert np.array_equal(pos.cpu().numpy().astype(np.uint64), np.concatenate(wpos))
    del t
    _free()


def test_c3_protein_1GiB(sm):
    spec = synth.text_spec("c3")
    t = synth.gen_text_device(spec, 0, spec.n)
    a = t.cpu().numpy()
    pats = synth.patterns("c3", spec=spec)
    assert len(pats) == 7 * 120
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch([p.data for p in pats], t, d)
    got = d.cpu().numpy()
    assert all(got[i] >= 1 for i, p in enumerate(pats) if p.kind == "sampled")
    idx = []
    for m in synth.PATTERN_LENGTHS["c3"]:
        idx += [i for i, p in enumerate(pats) if p.m == m and p.kind == "sampled"][:1]
        idx += [i for i, p in enumerate(pats) if p.m == m and p.kind == "random"][:1]
    with _pool() as ex:
        want = list(ex.map(lambda i: oracle.naive_count(pats[i].data, a), idx))
    assert [int(got[i]) for i in idx] == want
    del t
    _free()


def test_c4_binary_4GiB_properties(sm):
    spec = synth.text_spec("c4")
    t = synth.gen_text_device(spec, 0, spec.n)
    n = spec.n
    # sum over ALL 2^k patterns of length k over {0,1} = n - k + 1 (every alignment matches one)
    for k in (1, 8):
        allp = [bytes((v >> (k - 1 - j)) & 1 for j in range(k)) for v in range(1 << k)]
        d = torch.zeros(len(allp), dtype=torch.int64, device="cuda")
        sm.sm_count_batch(allp, t, d)
        assert int(d.sum().item()) == n - k + 1
    h = sm.sm_histogram(t).cpu().numpy()
    assert int(h[0]) + int(h[1]) == n
    pats = synth.patterns("c4", spec=spec)
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch([p.data for p in pats], t, d)
    got = d.cpu().numpy()
    assert (got >= 1).all()
    # element-wise on a 64 MiB prefix (count of p in t[:L] via max_alignments)
    L = 64 << 20
    a = t[:L].cpu().numpy()
    sel = [i for m in synth.PATTERN_LENGTHS["c4"] for i in [j for j, p in enumerate(pats) if p.m == m][:1]]
    d2 = torch.zeros(len(sel), dtype=torch.int64, device="cuda")
    sm.sm_count_batch([pats[i].data for i in sel], t, d2, max_alignments=L - 1024 + 1)
    with _pool() as ex:
        want = list(ex.map(lambda i: oracle.naive_count(pats[i].data, a[: L - 1024 + pats[i].m]), sel))
    assert d2.cpu().tolist() == want
    del t
    _free()


def test_c4_periodic_closed_forms(sm):
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))
    spec = synth.text_spec("c4p")
    assert spec.n == g["n"]
    t = synth.gen_text_device(spec, 0, spec.n)
    pats = [b"a" * c["m"] if c["p"].startswith("a^") and "b" not in c["p"] else b"a" * (c["m"] - 1) + b"b"
            for c in g["cases"]]
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch(pats, t, d)
    assert d.cpu().tolist() == [c["count"] for c in g["cases"]]
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


def test_c5_uniform_64GiB_shards(sm):
    from paper_1612_01506_b200 import dist
    spec = synth.text_spec("c5")
    N = spec.n
    free, _ = torch.cuda.mem_get_info()
    if free < N + (4 << 30):
        pytest.skip("needs 68 GiB of free device memory")
    t = synth.gen_text_device(spec, 0, N)
    pats = synth.patterns("c5", spec=spec, reader=lambda s, m: spec.substring(s, m))
    assert len(pats) == 200
    data = [p.data for p in pats]
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch(data, t, d)
    full = d.cpu().numpy()
    assert (full >= 1).all()  # includes the 28 boundary-straddling patterns per length
    # shard additivity: G = 2, 4, 8 ranks' owned counts sum to the 1-GPU count
    h = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
    for G in (2, 4, 8):
        tot = np.zeros(len(pats), dtype=np.int64)
        for sh in dist.all_shards(N, G, halo=63):
            c = dist.count_sharded(data, t[sh.own_lo: sh.held_hi], sh, hist=h)
            tot += c.cpu().numpy()
        assert np.array_equal(tot, full), G
    # oracle on windows around the boundary occurrences: the sampled occurrence is there
    for p in pats[:28]:
        lo = max(0, p.start - 4096)
        win = t[lo: p.start + p.m + 4096].cpu().numpy()
        assert oracle.naive_count(p.data, win) >= 1
    del t
    _free()
