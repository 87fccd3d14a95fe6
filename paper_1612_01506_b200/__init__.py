"""B200-native exact string matching (arXiv:1612.01506 hot path) -- Python binding.

Thin ctypes marshalling over the C ABI in ``include/smgpu.h`` (libsmgpu.so,
built in-tree for sm_100a).  Every step of the path on the text runs in the
library's CUDA kernels; this module only converts arguments.  There is no CPU
fallback: if the library or a CUDA device is missing, calls raise.

Names mirror the ABI:

* ``sm_count(p, t)``                      -> int
* ``sm_report(p, t, cap=None)``           -> (positions int64 CUDA tensor, total)
* ``sm_symbol_order(t, p)``               -> list[int]   (0-based pi)
* ``sm_histogram(t, out=None)``           -> int64[256] CUDA tensor (async)
* ``sm_order_from_histogram(hist, p)``    -> list[int]
* ``sm_count_async(p, t, d_count, ...)``  -> None (enqueued on the current stream)
* ``sm_count_batch(patterns, t, d_counts, ...)`` -> None (many patterns, few launches)
* ``sm_report_async(p, t, pos, d_count, ...)``
* ``sm_plan(p, hist, ...)``               -> (strategy, peel)

``t`` is a 1-D contiguous ``torch.uint8`` CUDA tensor (any storage offset).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SMGPU_LIB=debug selects the bounds-checked build (libsmgpu_debug.so, tests only);
# SMGPU_LIB=counters the compare-step instrumented build (libsmgpu_counters.so, NEXT-2)
# (SMGPU_LIB=/path/to/lib.so loads another build of the same ABI: A/B measurements in tools/)
_VARIANTS = {"debug": "libsmgpu_debug.so", "counters": "libsmgpu_counters.so"}
_SEL = os.environ.get("SMGPU_LIB", "")
LIB_PATH = _SEL if _SEL.endswith(".so") else os.path.join(_HERE, _VARIANTS.get(_SEL, "libsmgpu.so"))

SM_OK, SM_EINVAL, SM_ETRUNC, SM_ENOMEM, SM_ECUDA = 0, 1, 2, 3, 4
SM_STRATEGY_AUTO, SM_STRATEGY_FILTER, SM_STRATEGY_BLOCK, SM_STRATEGY_PACKED, SM_STRATEGY_PAIR = 0, 1, 2, 3, 4
SM_COUNT_ERROR = (1 << 64) - 1
SM_MAX_PATTERN = 4096
STRATEGY_NAMES = {1: "filter", 2: "block", 3: "packed1", 4: "packed2", 5: "pair", 6: "packed1-pre", 7: "packed2-pre"}

EXPORTED_SYMBOLS = (
    "sm_count", "sm_report", "sm_symbol_order", "sm_histogram", "sm_order_from_histogram",
    "sm_count_async", "sm_count_batch", "sm_count_batch_ordered", "sm_count_batch_multicast", "sm_report_async", "sm_report_batch", "sm_heuristic_order", "sm_plan", "sm_last_error", "sm_last_error_message",
    "sm_clear_error", "sm_status_string", "sm_version", "sm_launch_count", "sm_counters", "sm_trim_scratch",
)
COUNTER_NAMES = ("warp_tiles", "blocks", "steps", "filter_chunks", "filter_queued", "filter_survivors",
                 "filter_verify", "alpha_eff")


class SmError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{_status_name(status)}: {message}")
        self.status = status


def _status_name(s: int) -> str:
    return {0: "SM_OK", 1: "SM_EINVAL", 2: "SM_ETRUNC", 3: "SM_ENOMEM", 4: "SM_ECUDA"}.get(s, f"SM_{s}")


_lib = None
_u8p = ctypes.c_void_p
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t


def load_library(path: str = LIB_PATH):
    """Load libsmgpu.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    lib.sm_count.restype = ctypes.c_uint64
    lib.sm_count.argtypes = [_u8p, _sz, _u8p, _sz]
    lib.sm_report.restype = ctypes.c_int
    lib.sm_report.argtypes = [_u8p, _sz, _u8p, _sz, _vp, _sz, ctypes.POINTER(ctypes.c_uint64)]
    lib.sm_symbol_order.restype = ctypes.c_int
    lib.sm_symbol_order.argtypes = [_u8p, _sz, _u8p, _sz, _vp]
    lib.sm_histogram.restype = ctypes.c_int
    lib.sm_histogram.argtypes = [_u8p, _sz, _vp, _vp]
    lib.sm_order_from_histogram.restype = ctypes.c_int
    lib.sm_order_from_histogram.argtypes = [_vp, _u8p, _sz, _vp]
    lib.sm_count_async.restype = ctypes.c_int
    lib.sm_count_async.argtypes = [_u8p, _sz, _u8p, _sz, _vp, _vp, ctypes.c_uint32, ctypes.c_int, _vp, _vp]
    lib.sm_count_batch.restype = ctypes.c_int
    lib.sm_count_batch.argtypes = [_vp, _vp, _sz, _u8p, _sz, _sz, _vp, ctypes.c_int, _vp, _vp]
    lib.sm_count_batch_ordered.restype = ctypes.c_int
    lib.sm_count_batch_ordered.argtypes = [_vp, _vp, _sz, _u8p, _sz, _sz, _vp, _vp, _vp, ctypes.c_int, _vp, _vp]
    lib.sm_count_batch_multicast.restype = ctypes.c_int
    lib.sm_count_batch_multicast.argtypes = [_vp, _vp, _sz, _u8p, _sz, _sz, _vp, ctypes.c_int, _vp, _vp]
    lib.sm_report_batch.restype = ctypes.c_int
    lib.sm_report_batch.argtypes = [_vp, _vp, _sz, _u8p, _sz, _sz, _vp, ctypes.c_int, _vp, _sz, _vp,
                                    ctypes.c_uint64, _vp]
    lib.sm_report_async.restype = ctypes.c_int
    lib.sm_report_async.argtypes = [_u8p, _sz, _u8p, _sz, _vp, _vp, ctypes.c_uint32, ctypes.c_int, _vp, _sz,
                                    _vp, _vp]
    lib.sm_heuristic_order.restype = ctypes.c_int
    lib.sm_heuristic_order.argtypes = [_u8p, _sz, ctypes.c_int, ctypes.c_uint8, _vp]
    lib.sm_plan.restype = ctypes.c_int
    lib.sm_plan.argtypes = [_u8p, _sz, _vp, _vp, ctypes.c_uint32, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                            ctypes.POINTER(ctypes.c_uint32)]
    lib.sm_last_error.restype = ctypes.c_int
    lib.sm_last_error.argtypes = []
    lib.sm_last_error_message.restype = ctypes.c_char_p
    lib.sm_last_error_message.argtypes = []
    lib.sm_clear_error.restype = None
    lib.sm_clear_error.argtypes = []
    lib.sm_status_string.restype = ctypes.c_char_p
    lib.sm_status_string.argtypes = [ctypes.c_int]
    lib.sm_version.restype = ctypes.c_char_p
    lib.sm_version.argtypes = []
    lib.sm_launch_count.restype = ctypes.c_uint64
    lib.sm_launch_count.argtypes = []
    lib.sm_counters.restype = ctypes.c_int
    lib.sm_counters.argtypes = [_vp, ctypes.c_int]
    _lib = lib
    return lib


def _raise(status: int):
    lib = load_library()
    raise SmError(status, lib.sm_last_error_message().decode(errors="replace"))


def _pattern(p) -> Tuple[ctypes.Array, int]:
    if isinstance(p, str):
        p = p.encode("latin-1")
    b = bytes(p) if not isinstance(p, np.ndarray) else np.ascontiguousarray(p, dtype=np.uint8).tobytes()
    buf = ctypes.create_string_buffer(b, max(len(b), 1))
    return buf, len(b)


def _text(t) -> Tuple[int, int]:
    """(device pointer, n) of a 1-D contiguous uint8 CUDA tensor."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("t must be a torch.uint8 CUDA tensor (device-resident text)")
    if t.dtype != torch.uint8 or t.dim() != 1 or not t.is_contiguous():
        raise TypeError("t must be a 1-D contiguous torch.uint8 tensor")
    return t.data_ptr(), t.numel()


def _stream(stream) -> int:
    import torch
    if stream is None:
        # torch's current stream of the current device; the raw-handle query avoids the
        # ~15 us of Python device bookkeeping in torch.cuda.current_stream() (host-bound
        # small calls, tools/host_overhead.py)
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        if raw is not None:
            return raw(torch._C._cuda_getDevice())
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _u64_host(a) -> Optional[np.ndarray]:
    if a is None:
        return None
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    a = np.asarray(a)
    if a.dtype != np.uint64:
        a = a.astype(np.uint64)
    return np.ascontiguousarray(a)


def _u32_host(a) -> Optional[np.ndarray]:
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _np_ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


# ----------------------------------------------------------------------------- north-star calls

def sm_count(p, t) -> int:
    """Number of overlapping occurrences of p in the device text t."""
    lib = load_library()
    pb, m = _pattern(p)
    tp, n = _text(t)
    import torch
    torch.cuda.current_stream().synchronize()  # text produced on torch's stream must be ready
    r = lib.sm_count(pb, m, tp, n)
    if r == SM_COUNT_ERROR:
        _raise(lib.sm_last_error())
    return int(r)


def sm_report(p, t, cap: Optional[int] = None):
    """Ascending 0-based positions.  Returns (positions, total).

    cap=None: two-call idiom, all positions returned.  With a cap smaller than
    the total the first `cap` positions are returned and total > len(positions).
    """
    import torch
    lib = load_library()
    pb, m = _pattern(p)
    tp, n = _text(t)
    torch.cuda.current_stream().synchronize()
    cnt = ctypes.c_uint64(0)
    if cap is None:
        s = lib.sm_report(pb, m, tp, n, None, 0, ctypes.byref(cnt))
        if s not in (SM_OK, SM_ETRUNC):
            _raise(s)
        cap = int(cnt.value)
    pos = torch.empty(max(cap, 1), dtype=torch.int64, device=t.device)
    s = lib.sm_report(pb, m, tp, n, pos.data_ptr() if cap > 0 else None, cap, ctypes.byref(cnt))
    if s not in (SM_OK, SM_ETRUNC):
        _raise(s)
    total = int(cnt.value)
    return pos[: min(total, cap)], total


def sm_symbol_order(t, p) -> list:
    """Rarest-first comparison order pi from the device histogram of t."""
    import torch
    lib = load_library()
    pb, m = _pattern(p)
    tp, n = _text(t)
    torch.cuda.current_stream().synchronize()
    out = np.zeros(max(m, 1), dtype=np.uint32)
    s = lib.sm_symbol_order(tp, n, pb, m, out.ctypes.data)
    if s != SM_OK:
        _raise(s)
    return out[:m].tolist()


# ----------------------------------------------------------------------------- building blocks

def sm_histogram(t, out=None, stream=None):
    """Device byte histogram of t into an int64[256] CUDA tensor (async on `stream`)."""
    import torch
    lib = load_library()
    tp, n = _text(t)
    if out is None:
        out = torch.empty(256, dtype=torch.int64, device=t.device)
    s = lib.sm_histogram(tp, n, out.data_ptr(), _stream(stream))
    if s != SM_OK:
        _raise(s)
    return out


def sm_order_from_histogram(hist, p) -> list:
    lib = load_library()
    h = _u64_host(hist)
    pb, m = _pattern(p)
    out = np.zeros(max(m, 1), dtype=np.uint32)
    s = lib.sm_order_from_histogram(h.ctypes.data, pb, m, out.ctypes.data)
    if s != SM_OK:
        _raise(s)
    return out[:m].tolist()


def sm_count_async(p, t, d_count, hist=None, order: Optional[Sequence[int]] = None, peel: int = 0,
                   strategy: int = SM_STRATEGY_AUTO, stream=None) -> None:
    """Enqueue the count of p in t into the 1-element int64 CUDA tensor (or pointer) d_count."""
    lib = load_library()
    pb, m = _pattern(p)
    tp, n = _text(t)
    h, o = _u64_host(hist), _u32_host(order)
    dptr = d_count if isinstance(d_count, int) else d_count.data_ptr()
    s = lib.sm_count_async(pb, m, tp, n, _np_ptr(h), _np_ptr(o), peel, strategy, dptr, _stream(stream))
    if s != SM_OK:
        _raise(s)


class PatternBatch:
    """Host-side packing of a list of patterns for sm_count_batch (reusable across calls)."""

    def __init__(self, patterns):
        self.data = [bytes(p) if not isinstance(p, str) else p.encode("latin-1") for p in patterns]
        self.P = len(self.data)
        self._bufs = [ctypes.create_string_buffer(d, max(len(d), 1)) for d in self.data]
        self.ptrs = (ctypes.c_void_p * max(self.P, 1))(*[ctypes.addressof(x) for x in self._bufs])
        self.lens = (ctypes.c_size_t * max(self.P, 1))(*[len(d) for d in self.data])


def sm_count_batch(patterns, t, d_counts, hist=None, max_alignments: Optional[int] = None,
                   strategy: int = SM_STRATEGY_AUTO, stream=None) -> None:
    """Enqueue the counts of all patterns (list or PatternBatch) into int64 CUDA tensor d_counts[P].

    max_alignments: count only alignments i < max_alignments (a shard's owned range)."""
    lib = load_library()
    pb = patterns if isinstance(patterns, PatternBatch) else PatternBatch(patterns)
    tp, n = _text(t)
    h = _u64_host(hist)
    lim = (1 << 64) - 1 if max_alignments is None else int(max_alignments)
    dptr = d_counts if isinstance(d_counts, int) else d_counts.data_ptr()
    s = lib.sm_count_batch(ctypes.addressof(pb.ptrs), ctypes.addressof(pb.lens), pb.P, tp, n, lim, _np_ptr(h),
                           strategy, dptr, _stream(stream))
    if s != SM_OK:
        _raise(s)


def sm_count_batch_ordered(patterns, t, d_counts, orders=None, peels=None, hist=None,
                           max_alignments: Optional[int] = None, strategy: int = SM_STRATEGY_AUTO,
                           stream=None) -> None:
    """sm_count_batch with per-pattern comparison orders (list of sequences, or None for
    rarest-first) and peeling factors (list of ints, 0 = auto) -- NEXT-2 ablations."""
    lib = load_library()
    pb = patterns if isinstance(patterns, PatternBatch) else PatternBatch(patterns)
    tp, n = _text(t)
    h = _u64_host(hist)
    o = None if orders is None else np.ascontiguousarray(np.concatenate(
        [np.asarray(x, dtype=np.uint32) for x in orders]) if pb.P else np.zeros(0, np.uint32), dtype=np.uint32)
    if o is not None and o.size != sum(len(d) for d in pb.data):
        raise ValueError("orders must hold len(p) entries per pattern")
    r = None if peels is None else np.ascontiguousarray(np.asarray(peels, dtype=np.uint32))
    lim = (1 << 64) - 1 if max_alignments is None else int(max_alignments)
    dptr = d_counts if isinstance(d_counts, int) else d_counts.data_ptr()
    s = lib.sm_count_batch_ordered(ctypes.addressof(pb.ptrs), ctypes.addressof(pb.lens), pb.P, tp, n, lim,
                                   _np_ptr(h), _np_ptr(o), _np_ptr(r), strategy, dptr, _stream(stream))
    if s != SM_OK:
        _raise(s)


def sm_count_batch_multicast(patterns, t, mc_counts: int, hist=None, max_alignments: Optional[int] = None,
                             strategy: int = SM_STRATEGY_AUTO, stream=None) -> None:
    """NEXT-4: counts with the all-reduce fused into the kernel (multimem.red on the NVLink
    multicast address mc_counts of a u64[P] buffer bound on every rank; see smgpu.h).
    The caller zeroes its copy and synchronises the group before and after."""
    lib = load_library()
    pb = patterns if isinstance(patterns, PatternBatch) else PatternBatch(patterns)
    tp, n = _text(t)
    h = _u64_host(hist)
    lim = (1 << 64) - 1 if max_alignments is None else int(max_alignments)
    s = lib.sm_count_batch_multicast(ctypes.addressof(pb.ptrs), ctypes.addressof(pb.lens), pb.P, tp, n, lim,
                                     _np_ptr(h), strategy, int(mc_counts), _stream(stream))
    if s != SM_OK:
        _raise(s)


def sm_report_batch(patterns, t, pos, d_counts, hist=None, max_alignments: Optional[int] = None,
                    strategy: int = SM_STRATEGY_AUTO, stream=None, position_offset: int = 0) -> None:
    """Enqueue reporting for all patterns: d_counts[P] totals, positions concatenated in pattern
    order into pos (int64 CUDA tensor, capacity pos.numel())."""
    lib = load_library()
    pb = patterns if isinstance(patterns, PatternBatch) else PatternBatch(patterns)
    tp, n = _text(t)
    h = _u64_host(hist)
    lim = (1 << 64) - 1 if max_alignments is None else int(max_alignments)
    cap = 0 if pos is None else pos.numel()
    pptr = None if pos is None else pos.data_ptr()
    s = lib.sm_report_batch(ctypes.addressof(pb.ptrs), ctypes.addressof(pb.lens), pb.P, tp, n, lim, _np_ptr(h),
                            strategy, pptr, cap, d_counts.data_ptr(), int(position_offset), _stream(stream))
    if s != SM_OK:
        _raise(s)


def sm_report_async(p, t, pos, d_count, hist=None, order: Optional[Sequence[int]] = None, peel: int = 0,
                    strategy: int = SM_STRATEGY_AUTO, stream=None) -> None:
    """Enqueue reporting: first min(count, pos.numel()) positions into pos, total into d_count."""
    lib = load_library()
    pb, m = _pattern(p)
    tp, n = _text(t)
    h, o = _u64_host(hist), _u32_host(order)
    cap = 0 if pos is None else pos.numel()
    pptr = None if pos is None else pos.data_ptr()
    dptr = d_count if isinstance(d_count, int) else d_count.data_ptr()
    s = lib.sm_report_async(pb, m, tp, n, _np_ptr(h), _np_ptr(o), peel, strategy, pptr, cap, dptr,
                            _stream(stream))
    if s != SM_OK:
        _raise(s)


SM_ORDER_IDENTITY, SM_ORDER_PI_H, SM_ORDER_PI_HS = 0, 1, 2


def sm_heuristic_order(p, kind: int, space: int = 0x20) -> list:
    """Fixed comparison orders of PAPER.md:184-186 (identity, pi_h, pi_hs), 0-based."""
    lib = load_library()
    pb, m = _pattern(p)
    out = np.zeros(max(m, 1), dtype=np.uint32)
    s = lib.sm_heuristic_order(pb, m, kind, space, out.ctypes.data)
    if s != SM_OK:
        _raise(s)
    return out[:m].tolist()


def sm_plan(p, hist, order=None, peel: int = 0, strategy: int = SM_STRATEGY_AUTO) -> Tuple[int, int]:
    lib = load_library()
    pb, m = _pattern(p)
    h, o = _u64_host(hist), _u32_host(order)
    so, ro = ctypes.c_int(0), ctypes.c_uint32(0)
    s = lib.sm_plan(pb, m, _np_ptr(h), _np_ptr(o), peel, strategy, ctypes.byref(so), ctypes.byref(ro))
    if s != SM_OK:
        _raise(s)
    return int(so.value), int(ro.value)


def sm_last_error() -> Tuple[int, str]:
    lib = load_library()
    return int(lib.sm_last_error()), lib.sm_last_error_message().decode(errors="replace")


def sm_launch_count() -> int:
    return int(load_library().sm_launch_count())


def sm_counters(reset: bool = False) -> dict:
    """Compare-step counters of the instrumented build (SMGPU_LIB=counters), see smgpu.h."""
    out = np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
    s = load_library().sm_counters(out.ctypes.data, int(reset))
    if s:
        _raise(s)
    return {k: int(v) for k, v in zip(COUNTER_NAMES, out)}


def sm_trim_scratch(keep_bytes: int = 0) -> None:
    """Hand the library's cached scratch memory on the current device back to the driver."""
    lib = load_library()
    lib.sm_trim_scratch.restype = ctypes.c_int
    lib.sm_trim_scratch.argtypes = [_sz]
    s = lib.sm_trim_scratch(int(keep_bytes))
    if s != SM_OK:
        _raise(s)


def sm_version() -> str:
    return load_library().sm_version().decode()
