"""Host-side checks of the seeded input generator (synth/) -- no method arithmetic."""
import numpy as np

import oracle
import synth


def test_fmix_scalar_vs_numpy():
    xs = np.array([0, 1, 2, 12345678901234567, 2 ** 64 - 1], dtype=np.uint64)
    got = synth._fmix64_np(xs.copy())
    for x, g in zip(xs.tolist(), got.tolist()):
        assert synth.fmix64(int(x)) == int(g)


def test_lut_counts():
    for cfg in ("c1", "c2", "c3", "c4", "c5"):
        spec = synth.text_spec(cfg, n=1 << 12)
        lut = spec.lut
        assert lut.size == 65536
        syms = set(np.unique(lut).tolist())
        assert syms == set(spec.symbols)


def test_zipf_space_most_frequent():
    spec = synth.text_spec("c2", n=1 << 20)
    t = spec.host()
    h = np.bincount(t, minlength=256)
    assert int(np.argmax(h)) == 0x20
    assert abs(h[0x20] / t.size - 0.235) < 0.01
    assert len(np.nonzero(h)[0]) == 96


def test_host_generation_chunk_invariance_and_byte_at():
    spec = synth.text_spec("c3", n=1 << 16)
    full = spec.host()
    assert full.size == 1 << 16
    for a, b in [(0, 1), (1, 5), (3, 70000 - 4000), (12345, 50000), (65535, 65536)]:
        b = min(b, spec.n)
        part = synth.gen_text_host(spec.key, spec.lut, a, b - a, chunk=997)
        assert np.array_equal(part, full[a:b])
    for i in (0, 1, 2, 3, 4, 999, 65535):
        assert spec.byte_at(i) == int(full[i])


def test_patterns_are_substrings():
    spec = synth.text_spec("c2", n=1 << 16)
    t = spec.host()
    pats = synth.patterns("c2", spec=spec, per_m=3, lengths=[2, 8, 64])
    assert len(pats) == 9
    for ps in pats:
        assert ps.data == t[ps.start: ps.start + ps.m].tobytes()
        assert oracle.naive_count(ps.data, t) >= 1


def test_c3_random_patterns_and_c4p():
    spec = synth.text_spec("c3", n=1 << 14)
    pats = synth.patterns("c3", spec=spec, per_m=2, lengths=[4, 8])
    kinds = [p.kind for p in pats]
    assert kinds.count("random") == 40 and kinds.count("sampled") == 4
    letters = set(spec.symbols)
    for p in pats:
        assert set(p.data) <= letters and len(p.data) == p.m
    pp = synth.patterns("c4p")
    assert [(p.m, p.kind) for p in pp][:2] == [(1, "periodic-match"), (1, "periodic-miss")]
    assert pp[1].data == b"b"


def test_c5_boundary_patterns():
    N = 1 << 20
    spec = synth.text_spec("c5", n=N)
    pats = synth.patterns("c5", spec=spec, lengths=[8], reader=lambda s, m: spec.substring(s, m))
    b = [p for p in pats if p.kind == "boundary"]
    assert len(b) == 28 and len(pats) == 50
    cuts = synth.c5_boundaries(N)
    assert {p.start for p in b} == {s for a in cuts for s in (a - 1, a - 4, a - 7, a)}
