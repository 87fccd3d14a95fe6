"""CPU oracle for the hot path of arXiv:1612.01506, TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path in ``paper_1612_01506_b200/`` and never imports it.

Functions (all plain C in ``oracle.c``, each citing its passage there):

* ``naive_count``   -- Alg. 1 Naive-search, PAPER.md:41-53 (the definition).
* ``naive_report``  -- Alg. 1 with "printing position i".
* ``hist``          -- symbol counts of the text.
* ``order``         -- rarest-first stable permutation pi.
* ``alg4_count``    -- Alg. 4 LP-Freq-SIMD-Naive-search with order pi and
                        peeling factor r, PAPER.md:151-174 (emulated SIMDcompare).
* ``pi_h``          -- fixed heuristic order.
* ``kmp_count``     -- independent Knuth-Morris-Pratt cross-check.

Pins: tests/test_oracle.py.  Parity pinned for every function above
(``pi_h`` only by its permutation property and the SPEC example).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()

_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, no vectorisation flags)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}.{threading.get_ident()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:  # first use from several threads at once (tools/make_golden.py): build once
        return _load_locked()


def _load_locked():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.oracle_naive_count.restype = ctypes.c_uint64
        lib.oracle_naive_count.argtypes = [_u8p, ctypes.c_size_t, _u8p, ctypes.c_size_t]
        lib.oracle_naive_report.restype = ctypes.c_uint64
        lib.oracle_naive_report.argtypes = [_u8p, ctypes.c_size_t, _u8p, ctypes.c_size_t, _u64p, ctypes.c_uint64]
        lib.oracle_hist.restype = None
        lib.oracle_hist.argtypes = [_u8p, ctypes.c_size_t, _u64p]
        lib.oracle_order.restype = None
        lib.oracle_order.argtypes = [_u64p, _u8p, ctypes.c_size_t, _u32p]
        lib.oracle_alg4_count.restype = ctypes.c_uint64
        lib.oracle_alg4_count.argtypes = [_u8p, ctypes.c_size_t, _u8p, ctypes.c_size_t, ctypes.c_uint,
                                          _u32p, ctypes.c_uint, _u64p, _u64p, ctypes.c_uint64]
        lib.oracle_alg4_steps.restype = ctypes.c_uint64
        lib.oracle_alg4_steps.argtypes = [_u8p, ctypes.c_size_t, _u8p, ctypes.c_size_t, ctypes.c_size_t,
                                          _u32p, ctypes.c_uint, _u64p]
        lib.oracle_pi_h.restype = None
        lib.oracle_pi_h.argtypes = [ctypes.c_size_t, _u32p]
        lib.oracle_kmp_count.restype = ctypes.c_uint64
        lib.oracle_kmp_count.argtypes = [_u8p, ctypes.c_size_t, _u8p, ctypes.c_size_t]
        _lib = lib
    return _lib


def _u8(buf) -> np.ndarray:
    if isinstance(buf, (bytes, bytearray, memoryview)):
        a = np.frombuffer(bytes(buf), dtype=np.uint8)
    else:
        a = np.ascontiguousarray(np.asarray(buf), dtype=np.uint8)
    if a.size == 0:
        a = np.zeros(1, dtype=np.uint8)[:0]
    return a


def _ptr(a: np.ndarray, typ=_u8p):
    if a.size == 0:
        # a valid non-NULL pointer that is never dereferenced (n == 0 / m == 0)
        return ctypes.cast(ctypes.c_void_p(1), typ)
    return a.ctypes.data_as(typ)


def naive_count(p, t) -> int:
    """Alg. 1: number of overlapping occurrences of p in t."""
    pa, ta = _u8(p), _u8(t)
    return int(_load().oracle_naive_count(_ptr(pa), pa.size, _ptr(ta), ta.size))


def naive_report(p, t, cap: int | None = None) -> np.ndarray:
    """Alg. 1 reporting version: ascending 0-based positions."""
    pa, ta = _u8(p), _u8(t)
    lib = _load()
    if cap is None:
        cap = int(lib.oracle_naive_count(_ptr(pa), pa.size, _ptr(ta), ta.size))
    out = np.zeros(max(cap, 1), dtype=np.uint64)
    total = int(lib.oracle_naive_report(_ptr(pa), pa.size, _ptr(ta), ta.size, _ptr(out, _u64p), cap))
    return out[: min(total, cap)]


def hist(t) -> np.ndarray:
    """hist[c] = #{x : t[x] = c}."""
    ta = _u8(t)
    out = np.zeros(256, dtype=np.uint64)
    _load().oracle_hist(_ptr(ta), ta.size, _ptr(out, _u64p))
    return out


def order(h, p) -> np.ndarray:
    """Rarest-first stable comparison order pi, 0-based (readings R10, R11)."""
    ha = np.ascontiguousarray(np.asarray(h, dtype=np.uint64))
    assert ha.size == 256
    pa = _u8(p)
    out = np.zeros(max(pa.size, 1), dtype=np.uint32)
    _load().oracle_order(_ptr(ha, _u64p), _ptr(pa), pa.size, _ptr(out, _u32p))
    return out[: pa.size]


def alg4_count(p, t, alpha: int = 32, pi: Sequence[int] | None = None, r: int = 2,
               report: bool = False):
    """Alg. 4 LP-Freq-SIMD-Naive-search with emulated SIMDcompare.

    Returns (count, n_simdcompare_calls[, positions]).
    """
    pa, ta = _u8(p), _u8(t)
    m = pa.size
    if pi is None:
        pi = np.arange(m, dtype=np.uint32)
    pia = np.ascontiguousarray(np.asarray(pi, dtype=np.uint32))
    if m == 0:
        pia = np.zeros(1, dtype=np.uint32)
    ncmp = ctypes.c_uint64(0)
    lib = _load()
    if report:
        cap = naive_count(pa, ta)
        out = np.zeros(max(cap, 1), dtype=np.uint64)
        c = int(lib.oracle_alg4_count(_ptr(pa), m, _ptr(ta), ta.size, alpha, _ptr(pia, _u32p), r,
                                      ctypes.byref(ncmp), _ptr(out, _u64p), cap))
        return c, int(ncmp.value), out[: min(c, cap)]
    c = int(lib.oracle_alg4_count(_ptr(pa), m, _ptr(ta), ta.size, alpha, _ptr(pia, _u32p), r,
                                  ctypes.byref(ncmp), None, 0))
    return c, int(ncmp.value)


def alg4_steps(p, t, alpha: int, pi: Sequence[int] | None = None, r: int = 1):
    """SIMDcompare calls and alpha-blocks of Alg. 4 for any alpha >= 1.

    Instrumentation for the NEXT-2 compare counters.  Returns (n_compares, n_blocks)."""
    pa, ta = _u8(p), _u8(t)
    m = pa.size
    if pi is None:
        pi = np.arange(m, dtype=np.uint32)
    pia = np.ascontiguousarray(np.asarray(pi, dtype=np.uint32))
    if m == 0:
        pia = np.zeros(1, dtype=np.uint32)
    nb = ctypes.c_uint64(0)
    c = int(_load().oracle_alg4_steps(_ptr(pa), m, _ptr(ta), ta.size, alpha, _ptr(pia, _u32p), r,
                                      ctypes.byref(nb)))
    return c, int(nb.value)


def pi_h(m: int) -> np.ndarray:
    """Fixed heuristic order pi_h, 0-based."""
    out = np.zeros(max(m, 1), dtype=np.uint32)
    _load().oracle_pi_h(m, _ptr(out, _u32p))
    return out[:m]


def kmp_count(p, t) -> int:
    """Independent KMP occurrence count (overlapping)."""
    pa, ta = _u8(p), _u8(t)
    return int(_load().oracle_kmp_count(_ptr(pa), pa.size, _ptr(ta), ta.size))
