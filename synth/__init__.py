"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the string-matching method: it only makes
texts and patterns.  Both sides (tests/oracle and the GPU path) consume the
bytes it produces; the host (numpy) and device (``synth/csrc/synth_gen.cu``)
implementations of the same counter-based generator are bit-identical
(tests/test_synth.py, tests/test_gpu_synth.py).

Generator: byte i of a text with key K is

    w   = fmix64(K + (i >> 2) * GAMMA)          # SplitMix64 finaliser
    u16 = (w >> (16 * (i & 3))) & 0xFFFF
    t[i] = LUT[u16]

where LUT (65536 entries) is the integer inverse CDF of the symbol
distribution: symbol s owns ``counts[s]`` consecutive entries, counts summing
to 65536 (largest-remainder rounding of the probabilities, every symbol of
positive probability gets >= 1 entry).

Configs (BASELINE.json ``configs``; stand-ins for the paper's corpora,
PAPER.md:191, which are not available here):

  c1  DNA-like          n = 2^20, {A,C,G,T} uniform, seed 0
  c2  English-like      n = 2^28, 96 symbols {\\n, 0x20..0x7E}, Zipf s=1.1, space rank 1, seed 1
  c3  protein-like      n = 2^30, 20 amino-acid letters, Dirichlet(1) frequencies, seed 2
  c4  binary            n = 2^32, {0x00, 0x01} uniform, seed 3   (+ periodic a^(2^30))
  c5  uniform-256       N = 2^36 (sharded), all 256 byte values uniform, seed 4
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1

# ----------------------------------------------------------------------------
# scalar / vector SplitMix64 finaliser
# ----------------------------------------------------------------------------

def fmix64(z: int) -> int:
    z &= _MASK
    z = ((z ^ (z >> 30)) * _M1) & _MASK
    z = ((z ^ (z >> 27)) * _M2) & _MASK
    return z ^ (z >> 31)


def _fmix64_np(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z *= np.uint64(_M1)
    z ^= z >> np.uint64(27)
    z *= np.uint64(_M2)
    z ^= z >> np.uint64(31)
    return z


def stream_key(seed: int, stream: int) -> int:
    """Key of an independent stream (text = stream 0)."""
    return fmix64((seed * 0xD1B54A32D192ED03 + stream * GAMMA + 0x632BE59BD9B4E019) & _MASK)


def uniform_u64(seed: int, stream: int, k: int) -> int:
    """k-th 64-bit draw of stream (seed, stream)."""
    return fmix64((stream_key(seed, stream) + k * GAMMA) & _MASK)


# ----------------------------------------------------------------------------
# distributions -> 16-bit inverse-CDF lookup table
# ----------------------------------------------------------------------------

def lut_from_probs(symbols: List[int], probs: List[float]) -> np.ndarray:
    """Integer inverse CDF: symbol s gets counts[s] entries, sum 65536, each >= 1."""
    assert len(symbols) == len(probs) and len(symbols) >= 1
    p = np.asarray(probs, dtype=np.float64)
    p = p / p.sum()
    raw = p * 65536.0
    counts = np.maximum(np.floor(raw).astype(np.int64), 1)
    # largest remainder to reach exactly 65536
    diff = 65536 - int(counts.sum())
    rem = raw - np.floor(raw)
    idx = np.argsort(-rem, kind="stable")
    i = 0
    while diff > 0:
        counts[idx[i % len(idx)]] += 1
        diff -= 1
        i += 1
    while diff < 0:  # only when many symbols were lifted to 1
        j = int(np.argmax(counts))
        counts[j] -= 1
        diff += 1
    lut = np.repeat(np.asarray(symbols, dtype=np.uint8), counts)
    assert lut.size == 65536
    return lut


def _shuffle(seed: int, stream: int, items: List[int]) -> List[int]:
    """Fisher-Yates with the counter-based generator (deterministic)."""
    items = list(items)
    for k in range(len(items) - 1, 0, -1):
        j = uniform_u64(seed, stream, k) % (k + 1)
        items[k], items[j] = items[j], items[k]
    return items


def dist_uniform(symbols: List[int]):
    return symbols, [1.0] * len(symbols)


def dist_zipf_english(seed: int, s: float = 1.1):
    """96 printable symbols, Zipf(s); rank 1 = space (0x20), others shuffled."""
    others = [0x0A] + [c for c in range(0x21, 0x7F)]
    assert len(others) == 95
    ranked = [0x20] + _shuffle(seed, 77, others)
    probs = [1.0 / (r ** s) for r in range(1, 97)]
    return ranked, probs


def dist_dirichlet_protein(seed: int):
    """20 amino-acid letters, frequencies ~ Dirichlet(1) (normalised Exp(1) draws)."""
    letters = [ord(c) for c in "ACDEFGHIKLMNPQRSTVWY"]
    e = []
    for k in range(20):
        u = (uniform_u64(seed, 91, k) >> 11) * (1.0 / (1 << 53))  # [0,1)
        e.append(-math.log(1.0 - u))
    return letters, e


# ----------------------------------------------------------------------------
# host text generation (numpy)
# ----------------------------------------------------------------------------

def gen_text_host(key: int, lut: np.ndarray, start: int, length: int,
                  chunk: int = 1 << 24) -> np.ndarray:
    """Bytes [start, start+length) of the text with key `key` (host, numpy)."""
    out = np.empty(length, dtype=np.uint8)
    lut = np.asarray(lut, dtype=np.uint8)
    pos = 0
    while pos < length:
        a = start + pos
        b = min(start + length, a + chunk)
        w0, w1 = a >> 2, (b - 1) >> 2
        x = np.arange(w0, w1 + 1, dtype=np.uint64)
        z = np.uint64(key) + x * np.uint64(GAMMA)
        z = _fmix64_np(z)
        u16 = z.view(np.uint16)                 # little-endian: lane k = bits 16k..16k+15
        sym = lut[u16]
        off = a - (w0 << 2)
        out[pos: pos + (b - a)] = sym[off: off + (b - a)]
        pos += b - a
    return out


# ----------------------------------------------------------------------------
# configs
# ----------------------------------------------------------------------------

@dataclass
class TextSpec:
    name: str
    n: int
    seed: int
    symbols: List[int]
    probs: List[float]
    periodic: Optional[int] = None     # if set: t = byte^n (no generator)

    @property
    def key(self) -> int:
        return stream_key(self.seed, 0)

    @property
    def lut(self) -> np.ndarray:
        if not hasattr(self, "_lut"):
            self._lut = lut_from_probs(self.symbols, self.probs)
        return self._lut

    def host(self, start: int = 0, length: Optional[int] = None) -> np.ndarray:
        if length is None:
            length = self.n - start
        if self.periodic is not None:
            return np.full(length, self.periodic, dtype=np.uint8)
        return gen_text_host(self.key, self.lut, start, length)

    def byte_at(self, i: int) -> int:
        if self.periodic is not None:
            return self.periodic
        w = fmix64((self.key + (i >> 2) * GAMMA) & _MASK)
        return int(self.lut[(w >> (16 * (i & 3))) & 0xFFFF])

    def substring(self, start: int, m: int) -> bytes:
        return self.host(start, m).tobytes()


def text_spec(config: str, n: Optional[int] = None) -> TextSpec:
    c = config.lower()
    if c == "c1":
        sy, pr = dist_uniform([ord(ch) for ch in "ACGT"])
        return TextSpec("c1-dna", n or (1 << 20), 0, sy, pr)
    if c == "c2":
        sy, pr = dist_zipf_english(1)
        return TextSpec("c2-english-zipf", n or (1 << 28), 1, sy, pr)
    if c == "c3":
        sy, pr = dist_dirichlet_protein(2)
        return TextSpec("c3-protein-dirichlet", n or (1 << 30), 2, sy, pr)
    if c == "c4":
        sy, pr = dist_uniform([0, 1])
        return TextSpec("c4-binary", n or (1 << 32), 3, sy, pr)
    if c == "c4p":
        return TextSpec("c4-periodic", n or (1 << 30), 3, [0x61], [1.0], periodic=0x61)
    if c == "c5":
        sy, pr = dist_uniform(list(range(256)))
        return TextSpec("c5-uniform256", n or (1 << 36), 4, sy, pr)
    raise ValueError(config)


PATTERN_LENGTHS: Dict[str, List[int]] = {
    "c1": [4, 8, 16, 32],
    "c2": [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024],
    "c3": [4, 8, 16, 32, 64, 128, 256],
    "c4": [8, 32, 128, 512, 1024],
    "c4p": [1, 17, 1000],
    "c5": [8, 16, 32, 64],
}
PATTERNS_PER_M = {"c1": 50, "c2": 100, "c3": 100, "c4": 20, "c4p": 1, "c5": 50}


@dataclass
class PatternSpec:
    m: int
    start: Optional[int]       # sampled text position, or None for random/constructed
    kind: str                  # "sampled" | "random" | "periodic-match" | "periodic-miss" | "boundary"
    data: bytes = b""


def sample_start(spec: TextSpec, m: int, k: int, stream_base: int = 1000) -> int:
    """Uniform start position of the k-th sampled pattern of length m."""
    return uniform_u64(spec.seed, stream_base + m, k) % (spec.n - m + 1)


def patterns(config: str, spec: Optional[TextSpec] = None, per_m: Optional[int] = None,
             lengths: Optional[List[int]] = None,
             reader: Optional[Callable[[int, int], bytes]] = None) -> List[PatternSpec]:
    """The config's pattern set (BASELINE.json configs), deterministic.

    ``reader(start, m)`` returns text bytes (default: host generator)."""
    c = config.lower()
    spec = spec or text_spec(c)
    per_m = PATTERNS_PER_M[c] if per_m is None else per_m
    lengths = lengths or PATTERN_LENGTHS[c]
    rd = reader or spec.substring
    out: List[PatternSpec] = []
    if c == "c4p":
        for m in lengths:
            out.append(PatternSpec(m, None, "periodic-match", b"a" * m))
            out.append(PatternSpec(m, None, "periodic-miss", b"a" * (m - 1) + b"b"))
        return out
    for m in lengths:
        if m > spec.n:
            continue
        if c == "c5":
            out.extend(_c5_patterns(spec, m, per_m, rd))
            continue
        for k in range(per_m):
            s = sample_start(spec, m, k)
            out.append(PatternSpec(m, s, "sampled", rd(s, m)))
        if c == "c3":
            for k in range(20):
                data = bytes(spec.symbols[uniform_u64(spec.seed, 2000 + m, k * m + j) % len(spec.symbols)]
                             for j in range(m))
                out.append(PatternSpec(m, None, "random", data))
    return out


def c5_boundaries(N: int) -> List[int]:
    return [k * N // 8 for k in range(1, 8)]


def _c5_patterns(spec: TextSpec, m: int, per_m: int, rd) -> List[PatternSpec]:
    """28 boundary patterns (a_k-1, a_k-m//2, a_k-m+1, a_k for the 7 G=8 cuts) + uniform."""
    out = []
    for a in c5_boundaries(spec.n):
        for s in (a - 1, a - m // 2, a - m + 1, a):
            if 0 <= s <= spec.n - m:
                out.append(PatternSpec(m, s, "boundary", rd(s, m)))
    k = 0
    while len(out) < per_m:
        s = sample_start(spec, m, k)
        out.append(PatternSpec(m, s, "sampled", rd(s, m)))
        k += 1
    return out[:per_m]


# ----------------------------------------------------------------------------
# device generator (CUDA, bit-identical; test/bench infrastructure)
# ----------------------------------------------------------------------------
_HERE = os.path.dirname(os.path.abspath(__file__))
_CU = os.path.join(_HERE, "csrc", "synth_gen.cu")
_SO = os.path.join(_HERE, "libsmsynth.so")
_dlib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_CU):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-lineinfo",
                               "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, _CU])
        os.replace(tmp, _SO)
    return _SO


def _dev():
    global _dlib
    if _dlib is None:
        if not os.path.exists(_SO):
            raise RuntimeError(f"{_SO} missing: run synth.build() (nvcc)")
        lib = ctypes.CDLL(_SO)
        lib.synth_gen_text.restype = ctypes.c_int
        lib.synth_gen_text.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
        _dlib = lib
    return _dlib


def gen_text_device(spec: TextSpec, start: int, length: int, out=None, device=None):
    """Bytes [start, start+length) of `spec` generated on the GPU into a torch uint8 tensor."""
    import torch
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    if out is None:
        out = torch.empty(length, dtype=torch.uint8, device=dev)
    assert out.dtype == torch.uint8 and out.is_cuda and out.numel() >= length
    if length == 0:
        return out
    if spec.periodic is not None:
        out[:length].fill_(spec.periodic)
        return out
    lut = torch.from_numpy(spec.lut.copy()).to(dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = _dev().synth_gen_text(ctypes.c_void_p(out.data_ptr()), start, length, spec.key,
                               ctypes.c_void_p(lut.data_ptr()), ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"synth_gen_text failed: cuda error {rc}")
    torch.cuda.current_stream(dev).synchronize()
    return out
