"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Integer work throughout, so the bar is bit-exact: counts, positions, histograms
and orders must equal the oracle's.  Strategy, peeling factor r, comparison
order pi, tile size and the text's byte offset are free parameters that must
never change a result ("Clearly ... iff the k-bit of found is set":
AND is commutative, so any order/peeling gives Alg. 1's answer).
"""
import ctypes

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sm():
    import paper_1612_01506_b200 as sm
    sm.load_library()
    return sm


def dev(a: np.ndarray, offset: int = 0):
    """Device copy of host bytes `a`, placed at byte `offset` of a fresh allocation (unaligned views)."""
    buf = torch.empty(a.size + offset + 16, dtype=torch.uint8, device="cuda")
    buf.fill_(0xEE)
    if a.size:
        buf[offset: offset + a.size].copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return buf[offset: offset + a.size]


def count_async(sm, p, t, **kw):
    d = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    sm.sm_count_async(p, t, d, **kw)
    return int(d.item())


def report_async(sm, p, t, cap, **kw):
    d = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    pos = torch.full((max(cap, 1),), -7, dtype=torch.int64, device="cuda")
    sm.sm_report_async(p, t, pos[:cap] if cap else None, d, **kw)
    total = int(d.item())
    return pos[: min(cap, total)].cpu().numpy(), total


# ------------------------------------------------------------------------------------------- Fig. 1
def test_fig1(sm):
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig1.json")))
    t = dev(np.frombuffer(g["t"].encode(), dtype=np.uint8))
    p = g["p"].encode()
    assert sm.sm_count(p, t) == g["count"]
    pos, total = sm.sm_report(p, t)
    assert total == g["count"] and pos.cpu().tolist() == g["positions_0based"]
    assert sm.sm_symbol_order(t, p) == g["order_0based"]
    for strat in (1, 2, 4):
        for r in (1, 2, 3, 4):
            assert count_async(sm, p, t, strategy=strat, peel=r) == 1


# ------------------------------------------------------------------------------------------- closed forms
@pytest.mark.parametrize("n", [1, 15, 16, 17, 4096, 65537, 300000])
def test_periodic_closed_form(sm, n):
    t = dev(np.full(n, 0x61, dtype=np.uint8), offset=n % 7)
    for m in (1, 2, 17, 1000):
        for strat in (0, 1, 2, 4):
            want = max(n - m + 1, 0)
            assert count_async(sm, b"a" * m, t, strategy=strat) == want, (n, m, strat)
            assert count_async(sm, b"a" * (m - 1) + b"b", t, strategy=strat) == 0


def test_edge_cases(sm):
    t = dev(np.frombuffer(b"abcabcab", dtype=np.uint8))
    assert sm.sm_count(b"abcabcabc", t) == 0          # m > n
    assert sm.sm_count(b"abcabcab", t) == 1           # p = t
    empty = torch.empty(0, dtype=torch.uint8, device="cuda")
    assert sm.sm_count(b"a", empty) == 0              # n = 0
    pos, total = sm.sm_report(b"ab", t)
    assert total == 3 and pos.cpu().tolist() == [0, 3, 6]
    assert sm.sm_count(b"\x00", dev(np.zeros(33, dtype=np.uint8))) == 33   # NUL is a symbol


def test_maximum_pattern_length(sm):
    """m = SM_MAX_PATTERN (4096): the longest halo and table; every strategy, count and report."""
    M = sm.SM_MAX_PATTERN
    rng = np.random.default_rng(M)
    for sigma in (2, 4, 256):
        a = (rng.integers(0, sigma, (1 << 20) + 3, dtype=np.uint8) + (0x41 if sigma <= 4 else 0)).astype(np.uint8)
        a[200_000:200_000 + 3 * M] = np.tile(a[200_000:200_000 + M], 3)  # overlapping repeats -> several matches
        p = a[200_000:200_000 + M].tobytes()
        want = oracle.naive_count(p, a)
        assert want >= 3
        t = dev(a, 11)
        h = oracle.hist(a)
        for strat in ((0, 1, 2, 3, 4) if sigma <= 4 else (0, 1, 2, 4)):
            assert count_async(sm, p, t, hist=h, strategy=strat) == want, (sigma, strat)
        pos, total = sm.sm_report(p, t)
        assert total == want and pos.cpu().numpy().astype(np.uint64).tolist() == oracle.naive_report(p, a).tolist()


def test_errors(sm):
    t = dev(np.frombuffer(b"hello", dtype=np.uint8))
    with pytest.raises(sm.SmError) as e:
        sm.sm_count(b"", t)
    assert e.value.status == sm.SM_EINVAL
    with pytest.raises(sm.SmError):
        sm.sm_count(b"x" * (sm.SM_MAX_PATTERN + 1), dev(np.zeros(10000, dtype=np.uint8)))
    lib = sm.load_library()
    host = (ctypes.c_uint8 * 64)()
    r = lib.sm_count(b"ab", 2, ctypes.addressof(host), 64)   # host text: rejected, no CPU fallback
    assert r == sm.SM_COUNT_ERROR and lib.sm_last_error() == sm.SM_EINVAL
    with pytest.raises(sm.SmError):
        count_async(sm, b"ab", t, order=[0, 0])


# ------------------------------------------------------------------------------------------- histogram / order
@pytest.mark.parametrize("n,off", [(0, 0), (1, 3), (15, 1), (16, 0), (17, 15), (4099, 5), (1 << 20, 9), (3_000_001, 0)])
def test_histogram(sm, n, off):
    rng = np.random.default_rng(n + off)
    a = rng.integers(0, 256, n, dtype=np.uint8) if n % 2 else (rng.zipf(1.3, n) % 256).astype(np.uint8)
    t = dev(a, off)
    got = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
    assert np.array_equal(got, oracle.hist(a))


def test_symbol_order_matches_oracle(sm):
    spec = synth.text_spec("c2", n=1 << 18)
    a = spec.host()
    t = dev(a)
    h = oracle.hist(a)
    rng = np.random.default_rng(7)
    for m in (1, 2, 5, 64, 333, 1024, 4096):
        s = int(rng.integers(0, a.size - m))
        p = a[s:s + m].tobytes()
        want = oracle.order(h, p).tolist()
        assert sm.sm_symbol_order(t, p) == want
        assert sm.sm_order_from_histogram(h, p) == want


# ------------------------------------------------------------------------------------------- differential
def _case(rng):
    sigma = int(rng.choice([1, 2, 4, 20, 96, 256]))
    n = int(rng.choice([0, 1, 7, 16, 100, 1000, 4095, 4096, 4097, 20000, 65536, 70001]))
    n = max(0, n + int(rng.integers(-3, 4)))
    m = int(rng.choice([1, 2, 3, 4, 5, 8, 13, 16, 17, 31, 32, 64, 100, 255, 1024, 4096]))
    a = rng.integers(0, sigma, n, dtype=np.uint8) + int(rng.integers(0, 256 - sigma + 1))
    a = a.astype(np.uint8)
    if n >= m and rng.random() < 0.75:
        s = int(rng.integers(0, n - m + 1))
        p = a[s:s + m].tobytes()
    else:
        p = (rng.integers(0, sigma, m) + (a[0] if n else 0)).astype(np.uint8).tobytes()
    return a, p


def test_random_differential_count(sm):
    rng = np.random.default_rng(1234)
    for trial in range(600):
        a, p = _case(rng)
        m = len(p)
        off = int(rng.integers(0, 16))
        t = dev(a, off)
        want = oracle.naive_count(p, a)
        h = oracle.hist(a)
        strat = int(rng.choice([0, 1, 2, 4]))
        peel = int(rng.integers(0, m + 2))
        order = rng.permutation(m).tolist() if rng.random() < 0.4 else None
        got = count_async(sm, p, t, hist=h, order=order, peel=peel, strategy=strat)
        assert got == want, dict(trial=trial, n=a.size, m=m, off=off, strat=strat, peel=peel)


def test_random_differential_report(sm):
    rng = np.random.default_rng(99)
    for trial in range(250):
        a, p = _case(rng)
        off = int(rng.integers(0, 16))
        t = dev(a, off)
        want = oracle.naive_report(p, a)
        strat = int(rng.choice([0, 1, 2, 4]))
        order = rng.permutation(len(p)).tolist() if rng.random() < 0.3 else None
        pos, total = report_async(sm, p, t, cap=want.size + 3, hist=oracle.hist(a), order=order, strategy=strat)
        assert total == want.size
        assert pos.astype(np.uint64).tolist() == want.tolist(), dict(trial=trial, n=a.size, m=len(p), strat=strat)


def test_report_truncation(sm):
    a = np.frombuffer(b"ab" * 5000, dtype=np.uint8)
    t = dev(a)
    want = oracle.naive_report(b"ab", a)
    for strat in (1, 2, 4):
        pos, total = report_async(sm, b"ab", t, cap=100, strategy=strat)
        assert total == 5000 and pos.tolist() == want[:100].tolist()
    pos, total = sm.sm_report(b"ab", t, cap=7)
    assert total == 5000 and pos.cpu().tolist() == want[:7].tolist()
    lib = sm.load_library()
    assert lib.sm_last_error() == sm.SM_ETRUNC


@pytest.mark.parametrize("cap", [(1 << 20) + 17, 512 * 3000 + 34, 10])
def test_report_truncated_dense_1gib(sm, cap):
    """A truncated report of an everywhere-matching pattern on a 1 GiB text: the staged records
    overflow the default staging pool (its last chunk partial, cap % 512 in 1..34 or tiny), so the
    overflow pass and the chunk terminators are exercised.  Expected values are
    the closed form of a^n / a^m (every alignment matches; pinned in tests/test_oracle.py)."""
    n, m = 1 << 30, 17
    t = torch.full((n,), 0x61, dtype=torch.uint8, device="cuda")
    d = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    pos = torch.full((cap,), -7, dtype=torch.int64, device="cuda")
    sm.sm_report_async(b"a" * m, t, pos, d)
    assert int(d.item()) == n - m + 1
    assert torch.equal(pos, torch.arange(cap, dtype=torch.int64, device="cuda"))
    del t, pos
    torch.cuda.empty_cache()


def test_dense_report_every_alignment(sm):
    n = 300_003
    t = dev(np.full(n, 7, dtype=np.uint8), 3)
    for m, strat in ((1, 2), (3, 2), (3, 1), (3, 4), (1, 4)):
        pos, total = report_async(sm, bytes([7]) * m, t, cap=n, strategy=strat)
        assert total == n - m + 1
        assert np.array_equal(pos, np.arange(n - m + 1))


# ------------------------------------------------------------------------------------------- seams
def test_tile_seams(sm):
    """Occurrences planted across every tile / chunk / warp boundary, for both tile sizes."""
    rng = np.random.default_rng(5)
    for n in (64 * 4096 - 5, 600 * 16384 + 11):
        a = rng.integers(0, 200, n, dtype=np.uint8)
        for m in (2, 16, 33, 700):
            p = (rng.integers(200, 256, m)).astype(np.uint8)
            b = a.copy()
            starts = []
            for T in (4096, 16384):
                for k in range(1, n // T):
                    for d in (-m + 1, -m // 2, -1, 0, 1):
                        s = k * T + d
                        if 0 <= s <= n - m:
                            starts.append(s)
            starts = sorted(set(starts))[:: max(1, len(starts) // 400)]
            kept = []
            for s in starts:          # keep planted copies non-overlapping
                if not kept or s >= kept[-1] + m:
                    b[s:s + m] = p
                    kept.append(s)
            for off in (0, 5):
                t = dev(b, off)
                want = oracle.naive_count(p.tobytes(), b)
                assert want >= len(kept)
                for strat in (1, 2, 4):
                    assert count_async(sm, p.tobytes(), t, strategy=strat) == want, (n, m, off, strat)


def test_boundary_residues(sm):
    """n - m + 1 at every residue mod 16 and around tile sizes; matches at the very end."""
    rng = np.random.default_rng(11)
    for base in (32, 4096, 16384 * 300):
        for dn in range(0, 16):
            n = base + dn
            a = rng.integers(0, 4, n, dtype=np.uint8)
            for m in (1, 5, 16):
                p = a[n - m:].tobytes()      # occurrence ending at t[n-1]
                want = oracle.naive_count(p, a)
                t = dev(a, dn % 3)
                for strat in (1, 2, 4):
                    assert count_async(sm, p, t, strategy=strat) == want


# ------------------------------------------------------------------------------------------- virtual shards
def test_virtual_shards_sum(sm):
    from paper_1612_01506_b200 import dist
    spec = synth.text_spec("c5", n=(1 << 22) + 13)
    a = spec.host()
    t = dev(a)
    H = 63
    for m in (8, 16, 64):
        pats = [a[s:s + m].tobytes() for s in
                [x for cut in dist.shard_bounds(a.size, 8)[1:-1] for x in (cut - 1, cut - m // 2, cut - m + 1, cut)]]
        for p in pats[:12]:
            want = oracle.naive_count(p, a)
            for G in (1, 2, 3, 8):
                tot = 0
                for sh in dist.all_shards(a.size, G, H):
                    view = t[sh.own_lo: sh.own_lo + sh.view_len(m)]
                    tot += count_async(sm, p, view)
                assert tot == want, (m, G)


# ------------------------------------------------------------------------------------------- batched launches
def test_count_batch_matches_oracle(sm):
    rng = np.random.default_rng(77)
    for sigma, n in ((256, 300_001), (4, 200_003), (20, 1 << 20), (2, 70_000)):
        a = rng.integers(0, sigma, n, dtype=np.uint8)
        pats = []
        for m in (1, 2, 3, 5, 8, 17, 40, 64, 200, 1024, 3000):
            for _ in range(7):
                s = int(rng.integers(0, n - m + 1))
                pats.append(a[s:s + m].tobytes())
        pats.append(bytes([255]) * 9)          # absent symbol (sigma < 256)
        pats.append(a[:5].tobytes())
        pats.append(a[n - 7:].tobytes())
        h = oracle.hist(a)
        t = dev(a, 3)
        for lim in (None, n // 3, 1, 0):
            d = torch.full((len(pats),), -1, dtype=torch.int64, device="cuda")
            sm.sm_count_batch(pats, t, d, hist=h, max_alignments=lim)
            got = d.cpu().tolist()
            for i, p in enumerate(pats):
                view = a if lim is None else a[: min(n, lim + len(p) - 1)]
                assert got[i] == oracle.naive_count(p, view), (sigma, n, lim, i, len(p))


@pytest.mark.parametrize("lengths", [
    [8] * 32,                 # 256 table entries: the small parameter block
    [8] * 32 + [1],           # 257: the 2048-entry block
    [32] * 64,                # 2048
    [32] * 63 + [33],         # 2049: the 6400-entry block
    [100] * 64,               # 6400
    [100] * 64 + [7],         # 6407: two launches
])
def test_batch_table_capacity_boundaries(sm, lengths):
    """Launch parameter blocks come in three table capacities (256 / 2048 / 6400 entries,
    search_dispatch.cuh launch_cap); batches whose tables sit on either side of each bound
    must count and report exactly like the oracle (every strategy's launch path)."""
    rng = np.random.default_rng(len(lengths) * 1000 + sum(lengths))
    n = 200_003
    a = rng.integers(0, 4, n, dtype=np.uint8) + 65  # 'A'..'D': dense enough to report
    pats = []
    for m in lengths:
        s = int(rng.integers(0, n - m + 1))
        pats.append(a[s:s + m].tobytes())
    want = [oracle.naive_count(p, a) for p in pats]
    t = dev(a, 5)
    h = oracle.hist(a)
    for strat in (1, 2, 3, 4):
        d = torch.full((len(pats),), -1, dtype=torch.int64, device="cuda")
        sm.sm_count_batch(pats, t, d, hist=h, strategy=strat)
        assert d.cpu().tolist() == want, (strat, len(lengths))
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    pos = torch.empty(max(sum(want), 1), dtype=torch.int64, device="cuda")
    sm.sm_report_batch(pats, t, pos, d)
    assert d.cpu().tolist() == want
    wp = np.concatenate([oracle.naive_report(p, a) for p in pats]) if sum(want) else np.zeros(0, np.uint64)
    assert np.array_equal(pos[: sum(want)].cpu().numpy().astype(np.uint64), wp)


def test_count_batch_ordered_any_order_any_peel(sm):
    """sm_count_batch_ordered (NEXT-2: the paper's fixed orders and r on the batched path):
    every comparison order and peeling factor gives Alg. 1's count, for every
    strategy, on binary / DNA / protein-like / wide alphabets."""
    rng = np.random.default_rng(4242)
    for sigma, n in ((2, 150_001), (4, 200_003), (20, 250_007), (96, 300_001)):
        a = rng.integers(0, sigma, n, dtype=np.uint8) + (0x41 if sigma <= 96 else 0)
        pats, orders, peels = [], [], []
        for m in (1, 2, 3, 4, 7, 16, 33, 100):
            for kind in range(4):
                s = int(rng.integers(0, n - m + 1))
                p = a[s:s + m].tobytes()
                if kind == 0:
                    o = list(range(m))                                  # Alg. 1 / 2 (identity)
                elif kind == 1:
                    o = sm.sm_heuristic_order(p, sm.SM_ORDER_PI_H)      # pi_h
                elif kind == 2:
                    o = sm.sm_heuristic_order(p, sm.SM_ORDER_PI_HS)     # pi_hs
                else:
                    o = rng.permutation(m).tolist()                     # any permutation
                pats.append(p)
                orders.append(o)
                peels.append(int(rng.integers(0, m + 1)))               # 0 = auto, else 1..m
        want = [oracle.naive_count(p, a) for p in pats]
        t = dev(a, 7)
        h = oracle.hist(a)
        for strat in (0, 1, 2, 3, 4) if sigma <= 4 else (0, 1, 2, 4):  # forced PACKED needs <= 4 symbols
            d = torch.full((len(pats),), -1, dtype=torch.int64, device="cuda")
            sm.sm_count_batch_ordered(pats, t, d, orders=orders, peels=peels, hist=h, strategy=strat)
            assert d.cpu().tolist() == want, (sigma, strat)


def test_count_batch_strategies_agree(sm):
    spec = synth.text_spec("c2", n=(1 << 21) + 5)
    a = spec.host()
    t = dev(a, 1)
    pats = [p.data for p in synth.patterns("c2", spec=spec, per_m=4)]
    want = [oracle.naive_count(p, a) for p in pats]
    for strat in (0, 1, 2, 4):
        d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        sm.sm_count_batch(pats, t, d, strategy=strat)   # hist computed on the device
        assert d.cpu().tolist() == want, strat


def test_count_sharded_virtual(sm):
    from paper_1612_01506_b200 import dist
    spec = synth.text_spec("c5", n=(1 << 22) + 77)
    a = spec.host()
    t = dev(a)
    N = a.size
    h = oracle.hist(a)
    pats = []
    for m in (8, 16, 64):
        for cut in dist.shard_bounds(N, 8)[1:-1]:
            for s in (cut - 1, cut - m // 2, cut - m + 1, cut):
                pats.append(a[s:s + m].tobytes())
    want = [oracle.naive_count(p, a) for p in pats]
    for G in (1, 2, 8):
        tot = np.zeros(len(pats), dtype=np.int64)
        for sh in dist.all_shards(N, G, halo=63):
            c = dist.count_sharded(pats, t[sh.own_lo: sh.held_hi], sh, hist=h)
            tot += c.cpu().numpy()
        assert tot.tolist() == want, G


def test_report_batch_concatenated(sm):
    rng = np.random.default_rng(5150)
    for sigma, n in ((2, 100_001), (96, 400_003), (4, 1 << 20)):
        a = rng.integers(0, sigma, n, dtype=np.uint8)
        pats = []
        for m in (1, 2, 3, 7, 16, 40, 300):
            for _ in range(6):
                s = int(rng.integers(0, n - m + 1))
                pats.append(a[s:s + m].tobytes())
        t = dev(a, 7)
        want_pos = [oracle.naive_report(p, a) for p in pats]
        want_cnt = [w.size for w in want_pos]
        flat = np.concatenate(want_pos) if want_pos else np.zeros(0, np.uint64)
        for cap in (flat.size, flat.size // 3, 0):
            d = torch.full((len(pats),), -1, dtype=torch.int64, device="cuda")
            pos = torch.full((max(cap, 1),), -7, dtype=torch.int64, device="cuda")
            sm.sm_report_batch(pats, t, pos[:cap] if cap else None, d, hist=oracle.hist(a))
            assert d.cpu().tolist() == want_cnt
            assert pos[:cap].cpu().numpy().astype(np.uint64).tolist() == flat[:cap].tolist(), (sigma, cap)


# ------------------------------------------------------------------------------------------- PACKED (b-bit codes)
PACKED_ALPHABETS = [b"ACGT", b"\x00\x01", b"a", b"ab", b"\x10\x30", b"ACG", b"\x00\x40\x80\xc0"]


def test_packed_strategy_matches_oracle(sm):
    rng = np.random.default_rng(31337)
    for alpha in PACKED_ALPHABETS:
        syms = np.frombuffer(alpha, dtype=np.uint8)
        for n in (1, 15, 16, 17, 5000, 70001, 1 << 20):
            a = syms[rng.integers(0, syms.size, n)]
            h = oracle.hist(a)
            for m in (1, 2, 5, 16, 31, 64, 300):
                if m > n:
                    continue
                s = int(rng.integers(0, n - m + 1))
                p = a[s:s + m].tobytes()
                off = int(rng.integers(0, 16))
                t = dev(a, off)
                want = oracle.naive_count(p, a)
                peel = int(rng.integers(0, m + 1))
                assert count_async(sm, p, t, hist=h, strategy=sm.SM_STRATEGY_PACKED, peel=peel) == want, \
                    (alpha, n, m, off, peel)
                if n <= 70001:
                    pos, total = report_async(sm, p, t, cap=want + 1, hist=h, strategy=sm.SM_STRATEGY_PACKED)
                    assert total == want and pos.astype(np.uint64).tolist() == oracle.naive_report(p, a).tolist()


def test_packed_applicability(sm):
    a = np.frombuffer(b"ACGT" * 1000, dtype=np.uint8)
    h = oracle.hist(a)
    s, r = sm.sm_plan(b"ACGTACGTAC", h)
    assert s == 4                                  # AUTO picks 2-bit codes for DNA
    with pytest.raises(sm.SmError):                # 'N' is absent from the text: not packable
        sm.sm_plan(b"ACGN", h, strategy=sm.SM_STRATEGY_PACKED)
    b = np.frombuffer(bytes(range(5)) * 100, dtype=np.uint8)
    with pytest.raises(sm.SmError):                # 5 symbols > 4
        sm.sm_plan(b"\x00\x01", oracle.hist(b), strategy=sm.SM_STRATEGY_PACKED)
    c = np.frombuffer(b"\x00\x01" * 100, dtype=np.uint8)
    assert sm.sm_plan(b"\x01\x00\x01", oracle.hist(c))[0] == 3   # binary: 1-bit codes


def test_packed_batch_and_dense_report(sm):
    rng = np.random.default_rng(4)
    a = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, 3_000_017)]
    t = dev(a, 5)
    pats = [a[s:s + m].tobytes() for m in (1, 2, 4, 8, 12, 32, 100) for s in rng.integers(0, a.size - m, 5)]
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch(pats, t, d, strategy=sm.SM_STRATEGY_PACKED)
    want = [oracle.naive_count(p, a) for p in pats]
    assert d.cpu().tolist() == want
    sub = pats[:10]
    cap = sum(want[:10])
    pos = torch.zeros(cap, dtype=torch.int64, device="cuda")
    d2 = torch.zeros(10, dtype=torch.int64, device="cuda")
    sm.sm_report_batch(sub, t, pos, d2)  # AUTO -> PACKED
    assert np.array_equal(pos.cpu().numpy().astype(np.uint64), np.concatenate([oracle.naive_report(p, a) for p in sub]))


def test_ten_thousand_random_cases_batched(sm):
    """>= 10k (text, pattern) cases through the batched path, every strategy."""
    rng = np.random.default_rng(10_000)
    total = 0
    for trial in range(24):
        sigma = int(rng.choice([1, 2, 3, 4, 20, 96, 256]))
        n = int(rng.choice([100, 4096, 33_333, 200_001]))
        a = (rng.integers(0, sigma, n) + int(rng.integers(0, 256 - sigma + 1))).astype(np.uint8)
        pats = []
        for _ in range(450):
            m = int(rng.choice([1, 2, 3, 4, 6, 8, 13, 24, 40, 64, 100]))
            m = min(m, n)
            if rng.random() < 0.8:
                s = int(rng.integers(0, n - m + 1))
                pats.append(a[s:s + m].tobytes())
            else:
                pats.append(bytes(rng.choice(np.unique(a), m)))
        t = dev(a, int(rng.integers(0, 16)))
        h = oracle.hist(a)
        want = [oracle.naive_count(p, a) for p in pats]
        strats = [0, 1, 2, 4] + ([3] if np.unique(a).size <= 4 else [])
        for strat in strats:
            try:
                d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
                sm.sm_count_batch(pats, t, d, hist=h, strategy=strat)
            except sm.SmError:
                assert strat == 3   # PACKED refuses alphabets it cannot encode
                continue
            assert d.cpu().tolist() == want, (trial, sigma, n, strat)
            total += len(pats)
    assert total >= 10_000


def test_concurrent_streams(sm):
    """Re-entrancy: launches on different streams with different patterns / texts overlap
    freely (no __constant__ or global state in the library)."""
    rng = np.random.default_rng(8)
    texts = [rng.integers(0, s, 1_000_003, dtype=np.uint8) for s in (4, 20, 96, 256)]
    devs = [dev(a, i) for i, a in enumerate(texts)]
    torch.cuda.synchronize()  # texts were written on the default stream
    streams = [torch.cuda.Stream() for _ in texts]
    jobs = []
    for a, t, st in zip(texts, devs, streams):
        pats = [a[s:s + m].tobytes() for m in (2, 5, 9, 33, 300) for s in rng.integers(0, a.size - m, 4)]
        d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        jobs.append((a, pats, d))
        with torch.cuda.stream(st):
            for _ in range(3):
                sm.sm_count_batch(pats, t, d, hist=oracle.hist(a), stream=st)
    torch.cuda.synchronize()
    for a, pats, d in jobs:
        assert d.cpu().tolist() == [oracle.naive_count(p, a) for p in pats]


def test_concurrent_host_threads(sm):
    """Re-entrancy across HOST threads (smgpu.h "Concurrency"): four threads call the library at
    the same time (ctypes releases the GIL inside each call), each on its own stream with its own
    text -- count batches that histogram the text themselves (per-thread pinned read-back,
    per-thread launch tables and occupancy cache, the shared scratch pool), reports through the
    pool's staging buffers, and the synchronous sm_count on cudaStreamPerThread.  Every result
    equals the oracle's, and the thread-local status of one thread's failing call (m = 0) does
    not leak into another's."""
    import threading

    rng = np.random.default_rng(81)
    sigmas = (2, 4, 20, 256)
    texts = [rng.integers(0, s, 700_001 + 13 * i, dtype=np.uint8) for i, s in enumerate(sigmas)]
    devs = [dev(a, i) for i, a in enumerate(texts)]
    plan = []
    for a in texts:
        pats = [a[s:s + m].tobytes() for m in (1, 2, 3, 7, 16, 40, 257) for s in rng.integers(0, a.size - m, 3)]
        plan.append((pats, [oracle.naive_count(p, a) for p in pats],
                     oracle.naive_report(pats[9], a).astype(np.int64)))
    torch.cuda.synchronize()
    errors = []
    start = threading.Barrier(len(texts))

    def work(k):
        try:
            torch.cuda.set_device(0)
            a, t = texts[k], devs[k]
            pats, want, want_pos = plan[k]
            st = torch.cuda.Stream()
            start.wait()
            for it in range(6):
                with torch.cuda.stream(st):
                    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
                    sm.sm_count_batch(pats, t, d, stream=st)           # library histogram inside
                    pos, total = sm.sm_report(pats[9], t)               # cudaStreamPerThread, synchronous
                    got1 = sm.sm_count(pats[(it * 5) % len(pats)], t)
                    if k == it % len(texts):
                        with pytest.raises(Exception):
                            sm.sm_count(b"", t)                         # SM_EINVAL on this thread only
                st.synchronize()
                assert d.cpu().tolist() == want, (k, it)
                assert total == want_pos.size and np.array_equal(pos.cpu().numpy(), want_pos), (k, it)
                assert got1 == want[(it * 5) % len(pats)], (k, it)
        except BaseException as e:  # noqa: BLE001 -- reported by the main thread
            errors.append((k, repr(e)))
            try:
                start.abort()
            except Exception:
                pass

    threads = [threading.Thread(target=work, args=(k,)) for k in range(len(texts))]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=300)
    assert not any(th.is_alive() for th in threads), "a worker thread hung"
    assert not errors, errors


def test_report_sharded_virtual(sm):
    """NEXT-4: per-shard reports with global positions (position_offset), concatenated per
    pattern in rank order == the 1-GPU report."""
    from paper_1612_01506_b200 import dist
    rng = np.random.default_rng(64)
    a = rng.integers(0, 3, (1 << 20) + 123, dtype=np.uint8)
    t = dev(a)
    N = a.size
    h = oracle.hist(a)
    pats = [a[c - 3: c + 4].tobytes() for c in dist.shard_bounds(N, 8)[1:-1]] + [b"\x01\x02", a[:9].tobytes()]
    want_c = [oracle.naive_count(p, a) for p in pats]
    want = [oracle.naive_report(p, a).astype(np.int64) for p in pats]
    for G in (1, 2, 3, 8):
        per_rank = []
        for sh in dist.all_shards(N, G, halo=63):
            c, p = dist.report_sharded(pats, t[sh.own_lo: sh.held_hi], sh, hist=h)
            per_rank.append((c.cpu().numpy(), p.cpu().numpy()))
        tot = sum(c for c, _ in per_rank)
        assert tot.tolist() == want_c, G
        for k in range(len(pats)):
            segs = []
            for c, p in per_rank:
                s0 = int(c[:k].sum())
                segs.append(p[s0: s0 + int(c[k])])
            assert np.concatenate(segs).tolist() == want[k].tolist(), (G, k)


# ------------------------------------------------------------- advisory caller histogram
@pytest.mark.parametrize("n", [4100, 300_017])
def test_caller_histogram_is_advisory(sm, n):
    """PAPER.md:113 lets the frequencies come "from some relevant corpus": a caller
    histogram that is not t's must never change a result.  DNA text with a few 'N'
    bytes, counted with an ACGT-only histogram (which plans PACKED 2-bit codes with a
    shift under which 'N' aliases 'G'): every entry point, AUTO and forced PACKED,
    equals Alg. 1 (the device support check sends the PACKED launches to their
    byte-compare fallback)."""
    rng = np.random.default_rng(n)
    a = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, n)].copy()
    a[rng.integers(0, n, 40)] = ord("N")
    a[n - 1] = ord("N")                      # also in the ragged tail
    h_acgt = np.zeros(256, dtype=np.uint64)
    for c in b"ACGT":
        h_acgt[c] = n // 4
    plan = sm.sm_plan(b"GGGGGG", h_acgt)
    assert sm.STRATEGY_NAMES[plan[0]].startswith("packed")  # the hazard is real: PACKED planned
    for off in (0, 5):
        t = dev(a, off)
        pats = [b"G", b"GN", b"AG", b"ACG", b"GGGGGG", a[7:19].tobytes(), a[100:104].tobytes(), b"TTTT"]
        want = [oracle.naive_count(p, a) for p in pats]
        for strat in (0, 3):
            ok_pats = [p for p in pats if all(h_acgt[c] for c in p)] if strat == 3 else pats
            wk = [oracle.naive_count(p, a) for p in ok_pats]
            d = torch.zeros(len(ok_pats), dtype=torch.int64, device="cuda")
            sm.sm_count_batch(ok_pats, t, d, hist=h_acgt, strategy=strat)
            assert d.cpu().tolist() == wk, (off, strat)
            for p, w in zip(ok_pats, wk):
                assert count_async(sm, p, t, hist=h_acgt, strategy=strat) == w, (p, off, strat)
            cap = sum(wk)
            pos = torch.zeros(max(cap, 1), dtype=torch.int64, device="cuda")
            d2 = torch.zeros(len(ok_pats), dtype=torch.int64, device="cuda")
            if strat == 3:  # reporting checks t's own histogram: 5 symbols, PACKED inapplicable
                with pytest.raises(sm.SmError) as ei:
                    sm.sm_report_batch(ok_pats, t, pos[:cap], d2, hist=h_acgt, strategy=strat)
                assert ei.value.status == sm.SM_EINVAL
                continue
            sm.sm_report_batch(ok_pats, t, pos[:cap] if cap else None, d2, hist=h_acgt, strategy=strat)
            assert d2.cpu().tolist() == wk
            wp = np.concatenate([oracle.naive_report(p, a) for p in ok_pats])
            assert np.array_equal(pos[:cap].cpu().numpy().astype(np.uint64), wp.astype(np.uint64))
            for p, w in zip(ok_pats[:3], wk[:3]):
                got, total = report_async(sm, p, t, w, hist=h_acgt, strategy=strat)
                assert total == w and np.array_equal(got.astype(np.uint64), oracle.naive_report(p, a))
        # the histogram of t itself still selects PACKED and agrees
        d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        sm.sm_count_batch(pats, t, d, hist=oracle.hist(a))
        assert d.cpu().tolist() == want


def test_caller_histogram_matching_text_keeps_packed(sm):
    """With a caller histogram that IS t's, the guarded PACKED launches run (and the
    fallback launches exit at once): same counts as the library-computed histogram."""
    spec = synth.text_spec("c1")
    a = spec.host()
    t = dev(a)
    pats = [a[s:s + m].tobytes() for s, m in ((10, 4), (999, 8), (5000, 16), (77777, 32), (123, 1))]
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch(pats, t, d, hist=oracle.hist(a))
    d0 = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch(pats, t, d0)
    want = [oracle.naive_count(p, a) for p in pats]
    assert d.cpu().tolist() == want and d0.cpu().tolist() == want


def test_trim_scratch_then_report(sm):
    """sm_trim_scratch hands the cached scratch back; the next report re-allocates it and
    still equals the oracle (and a report right after another reuses the cached pool)."""
    rng = np.random.default_rng(5)
    a = np.frombuffer(b"ab ", dtype=np.uint8)[rng.integers(0, 3, 300_001)].copy()
    t = dev(a, 3)
    pats = [b"ab", b"a b", b" ", b"bba"]
    want = [oracle.naive_count(p, a) for p in pats]
    wp = np.concatenate([oracle.naive_report(p, a) for p in pats])
    for trim in (False, True, False):
        if trim:
            sm.sm_trim_scratch(0)
        pos = torch.zeros(int(sum(want)), dtype=torch.int64, device="cuda")
        d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        sm.sm_report_batch(pats, t, pos, d)
        assert d.cpu().tolist() == want
        assert np.array_equal(pos.cpu().numpy().astype(np.uint64), wp.astype(np.uint64))
