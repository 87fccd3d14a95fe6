"""Pins for the CPU oracle (oracle/) -- things other than the oracle itself.

Each pin is chosen so that a plausible slip in oracle.c (an off-by-one in the
alignment range, a wrong index t[i+j] vs t[i+j-1], non-overlapping counting,
an unstable sort, a dropped alpha lane) fails at least one test:

* the paper's worked example, Fig. 1          -> golden/fig1.json
* closed forms of Alg. 1 (a^n / a^m, absent symbol, m>n, n=0, period-2 text)
* brute force: sum over ALL patterns of length m of count = n-m+1
* an independent KMP count and a slice-equality count on random inputs
* numpy.bincount for the histogram; Python's stable ``sorted`` for pi
* Alg. 4 (any pi, any r, any alpha) == Alg. 1 ("Clearly ...")
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _slice_count(p: bytes, t: bytes) -> int:
    m, n = len(p), len(t)
    return sum(1 for i in range(n - m + 1) if t[i:i + m] == p) if m <= n else 0


def _slice_positions(p: bytes, t: bytes):
    m, n = len(p), len(t)
    return [i for i in range(n - m + 1) if t[i:i + m] == p] if m <= n else []


# --------------------------------------------------------------------------- Fig. 1
def test_fig1_worked_example():
    g = json.load(open(os.path.join(GOLD, "fig1.json")))
    t, p = g["t"].encode(), g["p"].encode()
    assert oracle.naive_count(p, t) == g["count"]
    assert oracle.naive_report(p, t).tolist() == g["positions_0based"]
    h = oracle.hist(t)
    assert oracle.order(h, p).tolist() == g["order_0based"]
    for alpha in (1, 8, 16, 32):
        c, _ = oracle.alg4_count(p, t, alpha=alpha, pi=g["order_0based"], r=2)
        assert c == g["count"]


def test_spec_small_examples():
    assert oracle.naive_count(b"a", b"a") == 1
    assert oracle.naive_report(b"aa", b"aaaa").tolist() == [0, 1, 2]     # overlapping (R3)
    assert oracle.naive_count(b"x", b"") == 0


# --------------------------------------------------------------------------- closed forms
@pytest.mark.parametrize("n,m", [(1, 1), (5, 1), (5, 5), (64, 17), (1000, 1), (1000, 999), (4096, 1000)])
def test_closed_form_periodic(n, m):
    t = b"a" * n
    assert oracle.naive_count(b"a" * m, t) == n - m + 1
    assert oracle.naive_count(b"a" * (m - 1) + b"b", t) == 0
    assert oracle.kmp_count(b"a" * m, t) == n - m + 1


def test_closed_form_periodic_golden_small_scale():
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))
    # the golden file's n is 2^30; the formula it encodes is checked at a small n here
    for c in g["cases"]:
        if c["count"]:
            assert c["count"] == g["n"] - c["m"] + 1
    n = 3000
    for m in (1, 17, 1000):
        assert oracle.naive_count(b"a" * m, b"a" * n) == n - m + 1


def test_closed_forms_misc():
    rng = np.random.default_rng(0)
    t = rng.integers(0, 4, 5000, dtype=np.uint8).tobytes()
    assert oracle.naive_count(b"\x00\x01\x07", t) == 0                  # absent symbol 7
    assert oracle.naive_count(t[:100] + b"x", t[:100]) == 0             # m > n
    assert oracle.naive_count(b"ab", b"") == 0                           # n = 0
    assert oracle.naive_count(t[:777], t[:777]) == 1                     # p = t
    h = oracle.hist(t)
    assert int(h.sum()) == len(t)
    for c in range(4):
        assert oracle.naive_count(bytes([c]), t) == int(h[c])           # m = 1 -> hist
    k, j = 300, 7
    assert oracle.naive_count(b"ab" * j, b"ab" * k) == k - j + 1         # period-2 text
    assert oracle.naive_count(b"ba" * j, b"ab" * k) == k - j


def test_nul_is_ordinary_symbol():
    t = b"\x00\x00\x01\x00\x00"
    assert oracle.naive_count(b"\x00\x00", t) == 2
    assert oracle.naive_report(b"\x00", t).tolist() == [0, 1, 3, 4]


# --------------------------------------------------------------------------- brute force
@pytest.mark.parametrize("sigma,n,m", [(2, 10, 1), (2, 10, 3), (3, 9, 2), (3, 8, 4), (2, 12, 4), (1, 6, 3)])
def test_bruteforce_all_patterns_sum(sigma, n, m):
    rng = np.random.default_rng(sigma * 100 + n * 10 + m)
    for _ in range(5):
        t = rng.integers(0, sigma, n, dtype=np.uint8).tobytes()
        total = 0
        for tup in itertools.product(range(sigma), repeat=m):
            p = bytes(tup)
            c = oracle.naive_count(p, t)
            assert c == _slice_count(p, t)
            assert c == oracle.kmp_count(p, t)
            total += c
        assert total == n - m + 1


def test_random_vs_kmp_and_slices():
    rng = np.random.default_rng(1)
    for trial in range(400):
        sigma = int(rng.choice([1, 2, 3, 4, 20, 96, 256]))
        n = int(rng.integers(0, 600))
        m = int(rng.integers(1, 40))
        t = rng.integers(0, sigma, n, dtype=np.uint8).tobytes()
        if n >= m and rng.random() < 0.7:
            s = int(rng.integers(0, n - m + 1))
            p = t[s:s + m]
        else:
            p = rng.integers(0, sigma, m, dtype=np.uint8).tobytes()
        c = oracle.naive_count(p, t)
        assert c == oracle.kmp_count(p, t) == _slice_count(p, t)
        pos = oracle.naive_report(p, t)
        assert pos.tolist() == _slice_positions(p, t)


def test_report_cap_truncates_in_order():
    t = b"abababab"
    full = oracle.naive_report(b"ab", t)
    assert full.tolist() == [0, 2, 4, 6]
    assert oracle.naive_report(b"ab", t, cap=2).tolist() == [0, 2]


# --------------------------------------------------------------------------- histogram / order
def test_hist_vs_bincount():
    rng = np.random.default_rng(2)
    for n in (0, 1, 17, 10000):
        t = rng.integers(0, 256, n, dtype=np.uint8)
        assert oracle.hist(t).tolist() == np.bincount(t, minlength=256).tolist()


def test_order_golden():
    g = json.load(open(os.path.join(GOLD, "orders.json")))
    for c in g["cases"]:
        h = np.zeros(256, dtype=np.uint64)
        for ch, v in c["counts"].items():
            h[ord(ch)] = v
        assert oracle.order(h, c["p"].encode()).tolist() == c["order_0based"], c


def test_order_vs_stable_sorted():
    rng = np.random.default_rng(3)
    for _ in range(300):
        m = int(rng.integers(1, 300))
        sigma = int(rng.choice([2, 4, 20, 256]))
        p = rng.integers(0, sigma, m, dtype=np.uint8)
        h = rng.integers(0, 50, 256).astype(np.uint64)
        got = oracle.order(h, p).tolist()
        want = sorted(range(m), key=lambda j: (int(h[p[j]]), j))
        assert got == want
        assert sorted(got) == list(range(m))
        keys = [int(h[p[j]]) for j in got]
        assert keys == sorted(keys)


# --------------------------------------------------------------------------- Alg. 4
def test_alg4_equals_alg1_any_order_any_r():
    rng = np.random.default_rng(4)
    for trial in range(300):
        sigma = int(rng.choice([1, 2, 4, 20, 256]))
        n = int(rng.integers(0, 300))
        m = int(rng.integers(1, 20))
        t = rng.integers(0, sigma, n, dtype=np.uint8).tobytes()
        if n >= m and rng.random() < 0.7:
            s = int(rng.integers(0, n - m + 1))
            p = t[s:s + m]
        else:
            p = rng.integers(0, sigma, m, dtype=np.uint8).tobytes()
        alpha = int(rng.choice([1, 3, 8, 16, 32, 64]))
        pi = rng.permutation(m).astype(np.uint32)
        r = int(rng.integers(1, m + 3))
        c, ncmp, pos = oracle.alg4_count(p, t, alpha=alpha, pi=pi, r=r, report=True)
        assert c == oracle.naive_count(p, t)
        assert pos.tolist() == oracle.naive_report(p, t).tolist()


def test_alg4_absent_symbol_compare_bound():
    # p contains a byte absent from t; freq order compares it first, so each block stops
    # after the r peeled compares: at most ceil((n-m+1)/alpha) * r SIMDcompare calls.
    rng = np.random.default_rng(5)
    t = rng.integers(0, 4, 4000, dtype=np.uint8).tobytes()
    p = b"\x01\x02\x09\x03"
    pi = oracle.order(oracle.hist(t), p)
    assert pi[0] == 2
    for alpha in (16, 32):
        for r in (1, 2, 3):
            c, ncmp = oracle.alg4_count(p, t, alpha=alpha, pi=pi, r=r)
            assert c == 0
            assert ncmp == -(-(len(t) - 4 + 1) // alpha) * r


# --------------------------------------------------------------------------- Alg. 4 compare counts (NEXT-2)
def test_alg4_steps_equals_alg4_compares_small_alpha():
    """oracle_alg4_steps (found as one flag per alignment, any alpha) executes exactly the
    SIMDcompare calls of oracle_alg4_count (found as a 64-bit mask, alpha <= 64)."""
    rng = np.random.default_rng(41)
    for trial in range(300):
        sigma = int(rng.choice([1, 2, 4, 20, 256]))
        n = int(rng.integers(0, 400))
        m = int(rng.integers(1, 20))
        t = rng.integers(0, sigma, n, dtype=np.uint8).tobytes()
        if n >= m and rng.random() < 0.7:
            s0 = int(rng.integers(0, n - m + 1))
            p = t[s0:s0 + m]
        else:
            p = rng.integers(0, sigma, m, dtype=np.uint8).tobytes()
        alpha = int(rng.choice([1, 3, 8, 16, 32, 64]))
        pi = rng.permutation(m).astype(np.uint32)
        r = int(rng.integers(1, m + 3))
        _, ncmp = oracle.alg4_count(p, t, alpha=alpha, pi=pi, r=r)
        steps, blocks = oracle.alg4_steps(p, t, alpha=alpha, pi=pi, r=r)
        assert steps == ncmp, dict(trial=trial)
        assert blocks == (-(-(n - m + 1) // alpha) if n >= m else 0)


def test_alg4_steps_closed_forms():
    # t = a^n, p = a^m: no alignment ever fails, every block runs all m compares
    for n, m, alpha in ((5000, 7, 512), (4096, 1, 4096), (9999, 33, 1000), (70, 70, 4096)):
        steps, blocks = oracle.alg4_steps(b"a" * m, b"a" * n, alpha=alpha, r=2)
        nb = -(-(n - m + 1) // alpha)
        assert blocks == nb and steps == nb * m
    # a symbol absent from t compared first: every block stops after the r peeled compares
    t = bytes(np.random.default_rng(3).integers(0, 4, 20000, dtype=np.uint8))
    p = bytes([1, 2, 9, 3, 0])
    pi = oracle.order(oracle.hist(t), p)
    for alpha in (100, 512, 4096):
        for r in (1, 2, 4):
            steps, blocks = oracle.alg4_steps(p, t, alpha=alpha, pi=pi, r=r)
            assert steps == -(-(len(t) - 5 + 1) // alpha) * r


def test_alg4_steps_alpha1_is_scalar_naive_compares():
    """alpha = 1, identity order, r = 1: the character comparisons of Alg. 1,
    counted by brute force -- the paper's compares-per-alignment statistic."""
    rng = np.random.default_rng(8)
    for trial in range(60):
        n = int(rng.integers(1, 200))
        m = int(rng.integers(1, 8))
        t = rng.integers(0, int(rng.choice([2, 3, 26])), n, dtype=np.uint8).tobytes()
        p = rng.integers(0, 3, m, dtype=np.uint8).tobytes()
        want = 0
        for i in range(n - m + 1):
            for j in range(m):
                want += 1
                if t[i + j] != p[j]:
                    break
        steps, blocks = oracle.alg4_steps(p, t, alpha=1, r=1)
        assert steps == want and blocks == max(0, n - m + 1)


# --------------------------------------------------------------------------- pi_h
def test_pi_h_golden_and_permutation():
    g = json.load(open(os.path.join(GOLD, "pi_h.json")))
    for c in g["cases"]:
        assert (oracle.pi_h(c["m"]) + 1).tolist() == c["order_1based"]
    for m in range(1, 257):
        assert sorted(oracle.pi_h(m).tolist()) == list(range(m))
