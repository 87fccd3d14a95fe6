"""CPU-side checks of the C ABI library: it loads, exports every symbol the header
declares, and its host-only logic (order from histogram, planning, argument
checking) behaves.  No compute call runs here (no GPU in this container)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sm():
    from paper_1612_01506_b200 import _build
    _build.build()
    import paper_1612_01506_b200 as sm
    sm.load_library()
    return sm


def header_functions():
    src = open(os.path.join(ROOT, "include", "smgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sm_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(sm):
    lib = sm.load_library()
    names = header_functions()
    assert "sm_count" in names and "sm_report" in names and "sm_symbol_order" in names
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(sm.EXPORTED_SYMBOLS) == names


def test_order_from_histogram_matches_oracle(sm):
    rng = np.random.default_rng(0)
    for _ in range(200):
        m = int(rng.integers(1, 2000))
        p = rng.integers(0, int(rng.choice([2, 4, 20, 256])), m, dtype=np.uint8).tobytes()
        h = rng.integers(0, int(rng.choice([3, 1000])), 256).astype(np.uint64)  # 3: many tied counts
        assert sm.sm_order_from_histogram(h, p) == oracle.order(h, p).tolist()


def test_plan_policy(sm):
    h = np.zeros(256, dtype=np.uint64)
    for c in b"ACGT":
        h[c] = 1000
    s, r = sm.sm_plan(b"ACGTACGTACGT", h)
    assert s == 4 and r == 5                             # DNA: PACKED (2-bit codes); alpha_eff = 512, 512*(1/4)^5 = 1/2
    h2 = np.ones(256, dtype=np.uint64)
    s, r = sm.sm_plan(b"hello world", h2)
    assert s == sm.SM_STRATEGY_FILTER and r == 2        # phase B peels pi(1) and pi(2)
    s, r = sm.sm_plan(b"ab", h2, strategy=sm.SM_STRATEGY_BLOCK, peel=7)
    assert s == sm.SM_STRATEGY_BLOCK and r == 2           # r <- min(r, m)  (reading R9)
    hz = np.zeros(256, dtype=np.uint64)
    hz[ord("a")] = 10
    s, r = sm.sm_plan(b"aab", hz)                         # 'b' absent -> frequency 0 -> compared first
    assert s == sm.SM_STRATEGY_FILTER


def test_plan_auto_rule(sm):
    """AUTO (abi.cu make_plan, profiles/strategy_pair_r1.md): h1 = 1-(1-f1)^16 is FILTER's chunk
    queue rate, h12 = 1-(1-f1 f2)^16 PAIR's (h1 for m = 1); BLOCK/PACKED if h12 > 0.5 (PAIR
    instead of BLOCK for m = 2, where the pair test is the match), else PAIR if m >= 2 and
    h1 > 0.2 (0.12 for m >= 32), else FILTER."""
    h = np.zeros(256, dtype=np.uint64)
    # 20 symbols 'A'..'T': two frequent (10 % each), the rest rare
    for i, c in enumerate(range(65, 85)):
        h[c] = 1000 if i < 2 else 444
    rare, freq = b"T", b"A"
    s, _ = sm.sm_plan(rare + freq * 3, h)          # f1 ~ 4.9 %: h1 ~ 0.55 > 0.12, h12 ~ 0.08 -> PAIR
    assert s == 5 and sm.STRATEGY_NAMES[s] == "pair"
    s, _ = sm.sm_plan(rare, h)                     # m = 1: h12 := h1 ~ 0.51 > 0.5 -> BLOCK
    assert s == sm.SM_STRATEGY_BLOCK
    h[ord("T")] = 10                               # a rare pi(1): h1 ~ 0.9 %: FILTER
    s, _ = sm.sm_plan(b"T" + freq * 3, h)
    assert s == sm.SM_STRATEGY_FILTER
    hb = np.zeros(256, dtype=np.uint64)
    for c in range(65, 71):                        # 6 symbols, 'A' and 'B' 45 % each
        hb[c] = 9000 if c < 67 else 500
    s, _ = sm.sm_plan(b"ABAB", hb)                 # h12 = 1-(1-0.2025)^16 ~ 0.97 > 0.5
    assert s == sm.SM_STRATEGY_BLOCK               # 6 symbols: no 2-bit code -> BLOCK
    s, _ = sm.sm_plan(b"AB", hb)                   # m = 2: the exact one-pass PAIR replaces BLOCK
    assert s == 5
    s, _ = sm.sm_plan(b"ABCDE", hb)                # pi(1), pi(2) = C, D (5 % each): h1 ~ 0.56 -> PAIR
    assert s == 5
    s, _ = sm.sm_plan(b"ABCDE", hb, strategy=sm.SM_STRATEGY_PAIR)
    assert s == 5                                  # forced
    s, _ = sm.sm_plan(b"A", hb, strategy=sm.SM_STRATEGY_PAIR)
    assert s == sm.SM_STRATEGY_FILTER              # PAIR needs pi(2): m = 1 runs FILTER


def test_multicast_count_argument_checks(sm):
    """sm_count_batch_multicast validates before touching the GPU (n = 0: no text check)."""
    lib = sm.load_library()
    pats = sm.PatternBatch([b"ab", b"c"])
    args = (ctypes.addressof(pats.ptrs), ctypes.addressof(pats.lens), pats.P, None, 0, 2 ** 64 - 1, None, 0)
    assert lib.sm_count_batch_multicast(*args, 0x1003, None) == sm.SM_EINVAL      # misaligned multicast address
    assert lib.sm_count_batch_multicast(*args[:7], 9, 0x1000, None) == sm.SM_EINVAL  # bad strategy
    assert lib.sm_count_batch_multicast(*args[:7], 0, None, None) == sm.SM_EINVAL    # NULL counts


def test_argument_errors_without_gpu(sm):
    lib = sm.load_library()
    host = (ctypes.c_uint8 * 8)()
    assert lib.sm_count(b"a", 0, ctypes.addressof(host), 8) == sm.SM_COUNT_ERROR
    assert lib.sm_last_error() == sm.SM_EINVAL
    assert lib.sm_count(b"a", 1, ctypes.addressof(host), 8) == sm.SM_COUNT_ERROR   # host text rejected
    assert lib.sm_last_error() == sm.SM_EINVAL
    assert lib.sm_count(b"a", 1, None, 8) == sm.SM_COUNT_ERROR
    lib.sm_clear_error()
    assert lib.sm_last_error() == sm.SM_OK
    assert lib.sm_status_string(2) == b"SM_ETRUNC"
    with pytest.raises(sm.SmError):
        sm.sm_plan(b"ab", np.ones(256), order=[1, 1])


def test_heuristic_orders_vs_oracle_pi_h(sm):
    for m in range(1, 300):
        p = bytes((j * 7) % 251 for j in range(m))
        assert sm.sm_heuristic_order(p, sm.SM_ORDER_PI_H) == oracle.pi_h(m).tolist()
        assert sm.sm_heuristic_order(p, sm.SM_ORDER_IDENTITY) == list(range(m))
    # pi_hs: spaces last; the rest follows pi_h over the non-space ranks
    p = b"ab cd e  fgh"
    o = sm.sm_heuristic_order(p, sm.SM_ORDER_PI_HS)
    spaces = [j for j, c in enumerate(p) if c == 0x20]
    assert o[len(o) - len(spaces):] == spaces and sorted(o) == list(range(len(p)))
    rest = [j for j, c in enumerate(p) if c != 0x20]
    assert o[: len(rest)] == [rest[i] for i in oracle.pi_h(len(rest)).tolist()]
    assert sm.sm_heuristic_order(b"    ", sm.SM_ORDER_PI_HS) == [0, 1, 2, 3]
    assert sm.sm_heuristic_order(b"ab", sm.SM_ORDER_PI_HS) == sm.sm_heuristic_order(b"ab", sm.SM_ORDER_PI_H)
