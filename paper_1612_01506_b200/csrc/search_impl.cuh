// search_impl.cuh -- the hot path: exact occurrence counting / reporting of
// patterns in a device-resident byte text, pattern symbols compared rarest-first
// with peeled first comparisons (Algs. 3-4), B200-native.
//
// Persistent CTAs (3 per SM): warp 8 is the TMA producer, warps 0..7 compare.
// A launch runs a batch of patterns; each pattern is a full pass over the text.
//   * A3 staging (the paper loads 16/32 unaligned bytes): tiles
//     of T = 32 KiB plus the pattern's halo are copied HBM -> shared memory with
//     1-D TMA bulk copies (cp.async.bulk, 16-B granules, L2 evict-first) into a
//     ring (2-3 stages) of mbarrier-guarded buffers.  Ragged 16-B ends of the text are
//     loaded byte-wise by the producer, so nothing outside t[0..n) is read.
//   * SIMDcompare becomes a packed-byte compare: a lane owns
//     chunks of 16 consecutive alignments held as 4 x u32 words, one flag bit
//     (0x80) per alignment -- the paper's `found`.
//   * FILTER: pi(1) (the rarest symbol) is tested over 16-byte
//     chunks; flagged chunks are ballot-compacted, then pi(1), pi(2) compared
//     exactly (peeling r = 2) and pi(3..m) verified per survivor with early exit.
//   * PAIR: FILTER whose chunk test covers pi(1) AND pi(2) (one zero-byte test on the
//     OR of the two XORs) -- the rarest-two-symbol filter, for frequent pi(1).
//   * BLOCK: Alg. 4 as written: r peeled compares without a test,
//     then the pi-ordered loop with a warp-uniform exit test (__any_sync).
//   * PACKED: BLOCK on 1- or 2-bit codes of the text bytes (small alphabets).
//   * A6: popcount -> warp reduce -> one u64 atomic per warp and pattern.
//   * A8: reporting stages each tile's matches (per-warp u16 lists / bitmaps) in one
//     text pass; positions are expanded after a scan of the per-(pattern, tile) counts.
#pragma once
#include "device_util.cuh"
#include "launch.h"
#include "search.cuh"

namespace smgpu {

namespace {

__device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------
// Packed-byte helpers for one lane-chunk of 16 alignments (4 x u32 flag words,
// 0x80 per surviving alignment: the sm_100a form of the paper's `found`).
// ---------------------------------------------------------------------------
struct Found4 {
  uint32_t f0, f1, f2, f3;
};

// 16 bytes starting at shared address base16 + sel (base16 16-B aligned, sel in 0..15):
// two conflict-free LDS.128 + funnel shifts -- SIMDcompare's unaligned load
// (PAPER.md:101 _mm_loadu_si128) on shared memory.  The word offset Q =
// (sel >> 2) & 3 is a template parameter (callers branch once per warp-uniform
// step, not once per chunk); sh = 8 * (sel & 3).
template <int Q>
__device__ __forceinline__ uint4 window16_q(const uint8_t* base16, uint32_t sh) {
  const uint4 lo = lds128(base16);
  const uint4 hi = lds128(base16 + 16);
  const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
  return make_uint4(byte_window(w[Q], w[Q + 1], sh), byte_window(w[Q + 1], w[Q + 2], sh),
                    byte_window(w[Q + 2], w[Q + 3], sh), byte_window(w[Q + 3], w[Q + 4], sh));
}

// y - 0x01010101 (the borrow term of the zero-byte test) as an IMAD, k = 1 opaque to the
// compiler: phase A's chunk tests are ALU-pipe bound (LOP3 / SHF / IADD3), the FMA pipe idles
// (FILTER c5 and PAIR c3 m = 16: ALU pipe 76-79 %; under the pool's sustained power cap the SM
// clock falls to ~1.5 GHz and the ALU pipe, not HBM, sets the rate)
__device__ __forceinline__ uint32_t borrow_fma(uint32_t y, uint32_t k1) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, 0xFEFEFEFF;" : "=r"(r) : "r"(y), "r"(k1));
  return r;
}

// found &= SIMDcompare(...) for the 16 alignments whose compared bytes are `w`
// (k1 = 1 opaque, see eq_flags_fma)
__device__ __forceinline__ void found_and_eq(Found4& F, const uint4 w, uint32_t bc, uint32_t k1) {
  F.f0 &= eq_flags_fma(w.x, bc, k1);
  F.f1 &= eq_flags_fma(w.y, bc, k1);
  F.f2 &= eq_flags_fma(w.z, bc, k1);
  F.f3 &= eq_flags_fma(w.w, bc, k1);
}

__device__ __forceinline__ Found4 found_all() { return Found4{0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u}; }

__device__ __forceinline__ Found4 found_from_mask16(uint32_t vmask) {
  return Found4{nibble_to_flags(vmask & 0xFu), nibble_to_flags((vmask >> 4) & 0xFu),
                nibble_to_flags((vmask >> 8) & 0xFu), nibble_to_flags((vmask >> 12) & 0xFu)};
}

__device__ __forceinline__ uint32_t found_any(const Found4& F) { return (F.f0 | F.f1 | F.f2 | F.f3) & 0x80808080u; }

// bits b in [0,16) with lo <= u0 + b < hi (tile-relative 32-bit coordinates)
__device__ __forceinline__ uint32_t range_mask16_rel(int32_t u0, int32_t lo, int32_t hi) {
  int32_t l = min(max(lo - u0, 0), 16), h = min(max(hi - u0, 0), 16);
  if (h <= l) return 0u;
  return ((1u << h) - 1u) & ~((1u << l) - 1u);
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, v, d);
    if (lane >= d) v += u;
  }
  return v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// A6: add a warp's popcount sum to its pattern's count (one u64 atomic).
// (The NVLS multicast reduction of multi-GPU counts is nvls_epilogue, run once per launch
// by the last CTA: an inline-asm multimem.red here, inside the work loop, is a convergent
// operation that made the compiler add reconvergence barriers throughout it, +7 %.)
__device__ __forceinline__ void count_add(const LaunchArgs&, uint64_t* out, uint32_t v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(out), (unsigned long long)v);
}

// Per-tile view of one pattern of the batch (read from the kernel parameters).
struct Pat {
  uint32_t m, r, a1, bc1, s2, bc2, pre;
  uint32_t r1;          // PACKED: leading peeled steps whose window is register-resident
  uint32_t lim;         // bytes of the tile's stage buffer that hold this pattern's data (stage_len)
  const uint32_t* tbl;  // this pattern's table in the kernel parameters (m entries, pi order; constant cache)
};

// Per-thread compare-step counters (search.cuh Counter); compiled to nothing unless
// SMGPU_COUNTERS (the instrumented libsmgpu_counters.so).  Warp-uniform counters are
// flushed from lane 0, per-lane ones from every lane.
struct Ctr {
#ifdef SMGPU_COUNTERS
  unsigned long long v[kCounters] = {};
  __device__ __forceinline__ void add(int i, unsigned long long x) { v[i] += x; }
  __device__ __forceinline__ void flush(unsigned long long* out, int lane) {
    if (!out) return;
    for (int i = 0; i < kCounters; ++i) {
      const bool uniform = i != kCtrSurvivors && i != kCtrVerify;
      if (i == kCtrAlphaEff) {
        if (lane == 0 && v[i]) atomicMax(out + i, v[i]);
      } else if (v[i] && (!uniform || lane == 0)) {
        atomicAdd(out + i, v[i]);
      }
    }
  }
#else
  __device__ __forceinline__ void add(int, unsigned long long) {}
  __device__ __forceinline__ void flush(unsigned long long*, int) {}
#endif
};

// ---------------------------------------------------------------------------
// This CTA's work items (pattern k, tile ti), in order: w = blockIdx.x + i * gridDim.x
// over the pattern-major item space; for kEpiWrite (reporting overflow pass) entries
// blockIdx.x + i * gridDim.x of the launch's overflow queue instead.
// ---------------------------------------------------------------------------
template <int EPI, int CAP>
struct WorkIter {
  uint64_t next = blockIdx.x;
  uint64_t end;
  uint32_t k = 0;
  __device__ __forceinline__ explicit WorkIter(const LaunchParams<CAP>& P)
      : end(EPI == kEpiWrite ? (uint64_t)*P.a.ovf_n : P.a.total_work) {}
  // (pattern, tile) of pattern-major work index w; w must not decrease between calls
  __device__ __forceinline__ void map(const LaunchParams<CAP>& P, uint64_t w, uint32_t& kk, uint64_t& ti) {
    while (w >= P.d[k].work_end) ++k;
    kk = k;
    ti = w - (P.d[k].work_end - P.d[k].ntiles);
    if (P.d[k].flags & 1u) ti = P.d[k].ntiles - 1 - ti;  // alternating scan direction
  }
  __device__ __forceinline__ bool advance(const LaunchParams<CAP>& P, uint32_t& kk, uint64_t& ti) {
    if (next >= end) return false;
    if (EPI == kEpiWrite) {
      const uint64_t item = P.a.ovf_items[next];
      uint32_t j = 0;
      while (j + 1 < P.a.npat && !(item >= P.d[j].item_base && item < P.d[j].item_base + P.d[j].ntiles)) ++j;
      SMGPU_DCHECK(item >= P.d[j].item_base && item < P.d[j].item_base + P.d[j].ntiles);
      kk = j;
      ti = item - P.d[j].item_base;
    } else {
      map(P, next, kk, ti);
    }
    next += gridDim.x;
    return true;
  }
};

// ---------------------------------------------------------------------------
// TMA producer (one thread): for every work item (pattern, tile) of this CTA,
// wait for a free stage, load the ragged 16-B ends of t byte-wise, then one
// cp.async.bulk for the aligned interior, completion counted on full[s].
// ---------------------------------------------------------------------------
// PRE: kPackedBPre -- tiles come from the code array (CB code bits per alignment).
// Work dispatch: statically round-robin (item = blockIdx.x + j gridDim.x), or, with
// a.work_ctr, fetched from a counter in the order CTAs become free -- which keeps the
// window of text being read at any moment narrow (TMA ring probe on 4 GiB: 7.48-7.51 vs
// 7.21-7.26 TB/s static, tools/probe_dyn.py).  The producer fetches and publishes the
// item in tix[stage] before arming the stage; consumers read it after the stage's wait.
template <int EPI, int CAP, bool PRE = false, int CB = 1>
__device__ void produce(const LaunchParams<CAP>& P, uint8_t* ring, uint64_t* full, uint64_t* empty,
                        uint4* tix) {
  const LaunchArgs& a = P.a;
  const uint64_t pol = a.l2_policy == 2 ? l2_policy_evict_last()
                       : a.l2_policy == 1 ? l2_policy_evict_normal() : l2_policy_evict_first();
  const int64_t tlo = (int64_t)a.delta, thi = (int64_t)(a.delta + a.n);
  uint32_t s = 0, ph = 0;  // stage and its use parity
  bool wrapped = false;
  WorkIter<EPI, CAP> items(P);
  const bool dyn = EPI != kEpiWrite && a.work_ctr != nullptr;
  uint32_t k;
  uint64_t ti;
  while (true) {
    uint64_t w = 0;
    if (dyn) {
      w = atomicAdd(a.work_ctr, 1ull);
      if (w >= a.total_work) break;
      items.map(P, w, k, ti);
    } else if (!items.advance(P, k, ti)) {
      break;
    }
    const PatDesc& d = P.d[k];
    if (wrapped) mbar_wait_sleep(&empty[s], ph ^ 1u);  // consumers released this stage's previous use
    if (dyn)  // published by the arrive below (release)
      tix[s] = make_uint4((uint32_t)w, k, (uint32_t)ti, (ti < d.edge_lo || ti >= d.edge_hi) ? 1u : 0u);
    uint8_t* buf = ring + (size_t)s * a.stage_stride;
    if (PRE) {  // the tile's codes: one bulk copy from the padded code array (16-B granules)
      const uint64_t lo = ((d.k_begin + ti) * a.tile * CB) / 8u;
      mbar_arrive_expect_tx(&full[s], d.stage_len);
      SMGPU_DCHECK((lo & 15u) == 0 && (d.stage_len & 15u) == 0 && d.stage_len <= a.stage_stride);
      tma_load_1d(buf, a.codes + lo, d.stage_len, &full[s], pol);
      if (++s == a.stages) {
        s = 0;
        ph ^= 1u;
        wrapped = true;
      }
      continue;
    }
    const int64_t lo = (int64_t)((d.k_begin + ti) * a.tile) - (int64_t)d.pre;
    const int64_t hi = lo + (int64_t)d.stage_len;
    const int64_t vlo = imax(lo, tlo), vhi = imin(hi, thi);
    uint32_t tx = 0;
    int64_t alo = 0;
    SMGPU_DCHECK(hi - lo <= (int64_t)a.stage_stride);
    if (vlo < vhi) {
      alo = (vlo + 15) & ~(int64_t)15;
      const int64_t ahi = vhi & ~(int64_t)15;
      SMGPU_DCHECK(vlo >= tlo && vhi <= thi);  // never a byte outside t[0..n)
      bool ragged = false;
      if (alo < ahi) {
        for (int64_t o = vlo; o < alo; ++o) { buf[o - lo] = ldg_u8_nc(a.base + o); ragged = true; }
        for (int64_t o = ahi; o < vhi; ++o) { buf[o - lo] = ldg_u8_nc(a.base + o); ragged = true; }
        tx = (uint32_t)(ahi - alo);
      } else {
        for (int64_t o = vlo; o < vhi; ++o) { buf[o - lo] = ldg_u8_nc(a.base + o); ragged = true; }
      }
      if (ragged) fence_proxy_async_smem();
    }
    mbar_arrive_expect_tx(&full[s], tx);
    SMGPU_DCHECK(tx == 0 || (alo >= tlo && alo + tx <= thi && alo - lo + tx <= (int64_t)d.stage_len));
    if (tx) tma_load_1d(buf + (alo - lo), a.base + alo, tx, &full[s], pol);
    if (++s == a.stages) {
      s = 0;
      ph ^= 1u;
      wrapped = true;
    }
  }
  if (dyn) {  // end of work: the next stage carries the sentinel (no bytes)
    if (wrapped) mbar_wait_sleep(&empty[s], ph ^ 1u);
    tix[s].x = kNoItem;
    mbar_arrive(&full[s]);
  }
}

// FILTER phase A: does any of the 16 pi(1)-bytes of a chunk equal p[pi(1)]?
// (borrow-based zero-byte test: exact as a whole-chunk predicate)
// (k1 = 1, see borrow_fma)
__device__ __forceinline__ bool chunk_hit(const uint4 v, uint32_t bc, uint32_t k1) {
  const uint32_t y0 = v.x ^ bc, y1 = v.y ^ bc, y2 = v.z ^ bc, y3 = v.w ^ bc;
  return (((borrow_fma(y0, k1) & ~y0) | (borrow_fma(y1, k1) & ~y1) | (borrow_fma(y2, k1) & ~y2) |
           (borrow_fma(y3, k1) & ~y3)) &
          0x80808080u) != 0;
}

// PAIR phase A: does some alignment of chunk c match BOTH pi(1) and pi(2)?  The byte
// (t[x + pi(1)] ^ p[pi(1)]) | (t[x + pi(2)] ^ p[pi(2)]) is zero iff alignment x matches
// both, so one borrow-based zero-byte test on the OR covers the two comparisons
// (exact as a whole-chunk predicate, like chunk_hit).  QA = word offset of pi(2)'s window.
// the pi(1) bytes and pi(2) bytes of chunk c's 16 alignments (see pair_hit)
template <int QA, bool WORD_ALIGNED>
__device__ __forceinline__ void pair_windows(const uint8_t* buf, uint32_t c, uint32_t pre, uint32_t s2, uint4& v1,
                                             uint4& v2) {
  v1 = lds128(buf + pre + 16u * c);
  if constexpr (WORD_ALIGNED) {  // pi(2)'s window starts on a word: no funnel shifts
    if constexpr (QA == 0) {
      v2 = lds128(buf + 16u * c + (s2 & ~15u));
    } else {
      const uint4 lo = lds128(buf + 16u * c + (s2 & ~15u));
      const uint4 hi = lds128(buf + 16u * c + (s2 & ~15u) + 16u);
      const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
      v2 = make_uint4(w[QA], w[QA + 1], w[QA + 2], w[QA + 3]);
    }
  } else {
    v2 = window16_q<QA>(buf + 16u * c + (s2 & ~15u), (s2 & 3u) * 8u);
  }
}

template <int QA, bool WORD_ALIGNED = false>
__device__ __forceinline__ bool pair_hit(const uint8_t* buf, uint32_t c, uint32_t pre, uint32_t s2, uint32_t bc1,
                                         uint32_t bc2, uint32_t k1) {
  uint4 v1, v2;
  pair_windows<QA, WORD_ALIGNED>(buf, c, pre, s2, v1, v2);
  const uint32_t y0 = (v1.x ^ bc1) | (v2.x ^ bc2), y1 = (v1.y ^ bc1) | (v2.y ^ bc2);
  const uint32_t y2 = (v1.z ^ bc1) | (v2.z ^ bc2), y3 = (v1.w ^ bc1) | (v2.w ^ bc2);
  return (((borrow_fma(y0, k1) & ~y0) | (borrow_fma(y1, k1) & ~y1) | (borrow_fma(y2, k1) & ~y2) |
           (borrow_fma(y3, k1) & ~y3)) &
          0x80808080u) != 0;
}

// 0x80-per-byte flag words -> one word, bit (8k + 7 - i) <-> alignment 4i + k
__device__ __forceinline__ uint32_t compress_found(const Found4& F) {
  return (F.f0 & 0x80808080u) | ((F.f1 & 0x80808080u) >> 1) | ((F.f2 & 0x80808080u) >> 2) |
         ((F.f3 & 0x80808080u) >> 3);
}
__device__ __forceinline__ uint32_t gbit_to_alignment(uint32_t p) { return 4u * (7u - (p & 7u)) + (p >> 3); }

// compressed found word -> 16-bit mask, bit (4i + k) <-> alignment 4i + k: byte k's
// bit 7 of (g << i) is alignment 4i + k; the multiply gathers the four bit-7s of a
// word into bits 28..31 (the shifted copies never overlap, so no carries)
__device__ __forceinline__ uint32_t g_to_mask16(uint32_t g) {
  uint32_t m16 = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) m16 |= ((((g << i) & 0x80808080u) * 0x00204081u) >> 28) << (4 * i);
  return m16;
}

// FILTER phase B for one queued chunk c: Alg. 4's peeled part with r = 2 on its
// 16 alignments -- exact packed-byte compares of pi(1) and pi(2) without a test
// in between.  Returns the compressed found word (bit
// (8k + 7 - i) <-> tile-relative alignment u = 16c + 4i + k) of the survivors.
// Q = word offset of pi(2)'s window (warp-uniform per pattern, compile time).
template <int Q>
__device__ __forceinline__ uint32_t filter_entry(const Pat& pt, const uint8_t* buf, uint32_t c, bool edge,
                                                 int32_t rlo, int32_t rhi) {
  Found4 F = edge ? found_from_mask16(range_mask16_rel((int32_t)(16u * c), rlo, rhi)) : found_all();
  const uint32_t k1 = 1u + (pt.m >> 31);
  found_and_eq(F, lds128(buf + pt.pre + 16u * c), pt.bc1, k1);  // pi(1)
  SMGPU_DCHECK(pt.m < 2 || 16u * c + (pt.s2 & ~15u) + 32u <= pt.lim);
  if (pt.m >= 2)                                               // pi(2)
    found_and_eq(F, window16_q<Q>(buf + 16u * c + (pt.s2 & ~15u), (pt.s2 & 3u) * 8u), pt.bc2, k1);
  return compress_found(F);
}

// pi(3..m) for the survivors of pi(1), pi(2) held by the lanes of a warp (g = 0 on
// lanes without), early exit at the first mismatch (Alg. 3's inner loop; any
// order gives the same result).  Each lane first checks its own
// survivors for pi(3..min(m, kLaneVerifyMaxM)) (at most 32 serial steps, with many
// survivors all lanes stay busy); survivors of long patterns still alive after
// that are finished by the whole warp, one at a time, 32 positions of pi per step.
__device__ __forceinline__ uint32_t verify_survivors(const Pat& pt, const uint8_t* buf, uint32_t c, uint32_t g,
                                                     int lane, Ctr& C) {
  const uint32_t qlane = pt.m < kLaneVerifyMaxM ? pt.m : kLaneVerifyMaxM;
  {
    uint32_t todo = g;
    const uint8_t* xb = buf + pt.pre + 16u * c - pt.a1;  // smem address of alignment u = 16c
    while (todo) {
      const uint32_t p = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint8_t* xp = xb + gbit_to_alignment(p);
      for (uint32_t q = 2; q < qlane; ++q) {
        const uint32_t e = pt.tbl[q];
        SMGPU_DCHECK((uint32_t)(xp - buf) + (e & 0xFFFFu) < pt.lim);
        C.add(kCtrVerify, 1);
        if (xp[e & 0xFFFFu] != (e >> 16)) {
          g &= ~(1u << p);
          break;
        }
      }
    }
  }
  if (pt.m <= kLaneVerifyMaxM) return g;
  uint32_t todo = __ballot_sync(0xFFFFFFFFu, g != 0);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    uint32_t gs = __shfl_sync(0xFFFFFFFFu, g, src);
    const uint32_t cs = __shfl_sync(0xFFFFFFFFu, c, src);
    uint32_t keep = gs;
    const uint8_t* xb = buf + pt.pre + 16u * cs - pt.a1;
    while (gs) {
      const uint32_t p = __ffs(gs) - 1;
      gs &= gs - 1;
      const uint8_t* xp = xb + gbit_to_alignment(p);
      for (uint32_t q0 = kLaneVerifyMaxM; q0 < pt.m; q0 += 32) {
        const uint32_t q = q0 + lane;
        bool mis = false;
        if (q < pt.m) {
          const uint32_t e = pt.tbl[q];
          SMGPU_DCHECK((uint32_t)(xp - buf) + (e & 0xFFFFu) < pt.lim);
          mis = xp[e & 0xFFFFu] != (e >> 16);
          C.add(kCtrVerify, 1);
        }
        if (__any_sync(0xFFFFFFFFu, mis)) {
          keep &= ~(1u << p);
          break;
        }
      }
    }
    if (lane == src) g = keep;
  }
  return g;
}

// IN_G: input is a compressed found word (FILTER/BLOCK), else a 16-bit mask.
template <bool IN_G = true>
struct WriteSink {
  uint64_t run;    // next output index of this warp
  int64_t pbase;   // 0-based position of u = 0
  uint64_t* pos;
  uint64_t cap;
  __device__ __forceinline__ void operator()(uint32_t c, uint32_t g, int lane) {
    add(16u * c, IN_G ? g_to_mask16(g) : g, lane);
  }
  // mask bit b <-> tile-relative alignment base_u + b (lanes in ascending base_u order)
  __device__ __forceinline__ void add(uint32_t base_u, uint32_t mk, int lane) {
    const uint32_t pc = __popc(mk);
    const uint32_t incl = warp_incl_scan(pc, lane);
    uint64_t idx = run + incl - pc;
    while (mk) {
      const uint32_t b = __ffs(mk) - 1;
      mk &= mk - 1;
      if (idx < cap) pos[idx] = (uint64_t)(pbase + (int64_t)(base_u + b));
      ++idx;
    }
    run += __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
};

// Reporting: one warp's matches of a tile, ascending, as tile-relative alignment
// offsets u = 16c + b (u16, T <= 32 KiB) in the warp's shared list; n counts all of
// them even when the list (kListCap entries) overflows.
template <bool IN_G>
struct AppendSink {
  uint16_t* list;
  uint32_t n = 0;
  __device__ __forceinline__ void operator()(uint32_t c, uint32_t g, int lane) {
    add(16u * c, IN_G ? g_to_mask16(g) : g, lane);
  }
  __device__ __forceinline__ void add(uint32_t base_u, uint32_t mk, int lane) {
    const uint32_t pc = __popc(mk);
    const uint32_t incl = warp_incl_scan(pc, lane);
    uint32_t idx = n + incl - pc;
    while (mk) {
      const uint32_t b = __ffs(mk) - 1;
      mk &= mk - 1;
      if (idx < (uint32_t)kListCap) list[idx] = (uint16_t)(base_u + b);
      ++idx;
    }
    n += __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
};

struct CountSink {
  uint32_t n = 0;
  __device__ __forceinline__ void operator()(uint32_t, uint32_t g, int) { n += __popc(g); }
};

// Phase B of a FILTER tile: drain the warp's queue 32 entries at a time, one chunk
// per lane, all lanes busy.
template <int Q, class Sink>
__device__ __forceinline__ void filter_drain(const Pat& pt, const uint8_t* buf, int lane, const uint16_t* qc,
                                             uint32_t qlen, bool edge, int32_t rlo, int32_t rhi, Sink& sink,
                                             Ctr& C) {
  for (uint32_t b0 = 0; b0 < qlen; b0 += 32) {
    const uint32_t i = b0 + lane;
    uint32_t c = 0, g = 0;
    if (i < qlen) {
      c = qc[i];
      g = filter_entry<Q>(pt, buf, c, edge, rlo, rhi);
      C.add(kCtrSurvivors, __popc(g));
    }
    if (pt.m >= 3) g = verify_survivors(pt, buf, c, g, lane, C);
    sink(c, g, lane);
  }
}

// One warp's share of a FILTER tile, in groups of kGroup chunk-rows: phase A
// ballot-compacts the chunks whose pi(1)-bytes contain p[pi(1)] into the warp's
// queue (ascending chunk order); phase B (filter_drain) verifies them.
// PA (PAIR strategy): phase A tests pi(1) and pi(2) together (pair_hit, pi(2)'s window
// class QA; WA: the window is word-aligned), so only chunks with a pi(1)&pi(2) survivor
// are queued -- for frequent pi(1).
template <int CPL, bool PA, int QA, class Sink, bool WA = false>
__device__ __forceinline__ void filter_tile_q(const Pat& pt, const uint8_t* buf, uint32_t cw0, int lane, uint16_t* qc,
                                              bool edge, int32_t rlo, int32_t rhi, Sink& sink, Ctr& C) {
  C.add(kCtrChunks, 32u * CPL);
  if constexpr (PA) {
    const uint32_t k1 = 1u + (pt.m >> 31);  // 1, opaque (eq_flags_fma)
    if (pt.m == 2) {  // warp-uniform: pi(1), pi(2) are the whole pattern, so the pair test of
                      // phase A, taken per byte, IS the match -- one pass, no queue, no phase B
#pragma unroll
      for (int it = 0; it < CPL; ++it) {
        const uint32_t c = cw0 + it * 32u + lane;
        SMGPU_DCHECK(pt.pre + 16u * c + 16u <= pt.lim && 16u * c + (pt.s2 & ~15u) + 32u <= pt.lim);
        uint4 v1, v2;
        pair_windows<QA, WA>(buf, c, pt.pre, pt.s2, v1, v2);
        Found4 F = edge ? found_from_mask16(range_mask16_rel((int32_t)(16u * c), rlo, rhi)) : found_all();
        F.f0 &= eq_flags_fma((v1.x ^ pt.bc1) | (v2.x ^ pt.bc2), 0u, k1);
        F.f1 &= eq_flags_fma((v1.y ^ pt.bc1) | (v2.y ^ pt.bc2), 0u, k1);
        F.f2 &= eq_flags_fma((v1.z ^ pt.bc1) | (v2.z ^ pt.bc2), 0u, k1);
        F.f3 &= eq_flags_fma((v1.w ^ pt.bc1) | (v2.w ^ pt.bc2), 0u, k1);
        const uint32_t g = compress_found(F);
        C.add(kCtrSurvivors, __popc(g));
        sink(c, g, lane);
      }
      return;
    }
  }
  constexpr int G = CPL < kGroup ? CPL : kGroup;
  const uint32_t k1 = 1u + (pt.m >> 31);  // 1 (pt.m < 2^31), opaque: see borrow_fma
#pragma unroll
  for (int g0 = 0; g0 < CPL; g0 += G) {
    uint32_t qlen = 0;
#pragma unroll
    for (int it = g0; it < g0 + G; ++it) {
      const uint32_t c = cw0 + it * 32u + lane;
      SMGPU_DCHECK(pt.pre + 16u * c + 16u <= pt.lim);
      bool hit;
      if constexpr (PA) hit = pair_hit<QA, WA>(buf, c, pt.pre, pt.s2, pt.bc1, pt.bc2, k1);
      else hit = chunk_hit(lds128(buf + pt.pre + 16u * c), pt.bc1, k1);
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, hit);
      if (hit) qc[qlen + __popc(bal & lanemask_lt())] = (uint16_t)c;
      qlen += __popc(bal);
    }
    C.add(kCtrQueued, qlen);
    __syncwarp();
    switch ((pt.s2 >> 2) & 3u) {  // warp-uniform
      case 0: filter_drain<0>(pt, buf, lane, qc, qlen, edge, rlo, rhi, sink, C); break;
      case 1: filter_drain<1>(pt, buf, lane, qc, qlen, edge, rlo, rhi, sink, C); break;
      case 2: filter_drain<2>(pt, buf, lane, qc, qlen, edge, rlo, rhi, sink, C); break;
      default: filter_drain<3>(pt, buf, lane, qc, qlen, edge, rlo, rhi, sink, C); break;
    }
    __syncwarp();
  }
}

template <int CPL, class Sink>
__device__ __forceinline__ void filter_tile(const Pat& pt, const uint8_t* buf, uint32_t cw0, int lane, uint16_t* qc,
                                            bool edge, int32_t rlo, int32_t rhi, Sink& sink, Ctr& C) {
  filter_tile_q<CPL, false, 0>(pt, buf, cw0, lane, qc, edge, rlo, rhi, sink, C);
}

template <int CPL, class Sink>
__device__ __forceinline__ void pair_tile(const Pat& pt, const uint8_t* buf, uint32_t cw0, int lane, uint16_t* qc,
                                          bool edge, int32_t rlo, int32_t rhi, Sink& sink, Ctr& C) {
  const bool wa = (pt.s2 & 3u) == 0;  // warp-uniform
  switch ((pt.s2 >> 2) & 3u) {  // warp-uniform
    case 0:
      if (wa) filter_tile_q<CPL, true, 0, Sink, true>(pt, buf, cw0, lane, qc, edge, rlo, rhi, sink, C);
      else filter_tile_q<CPL, true, 0>(pt, buf, cw0, lane, qc, edge, rlo, rhi, sink, C);
      break;
    case 1:
      if (wa) filter_tile_q<CPL, true, 1, Sink, true>(pt, buf, cw0, lane, qc, edge, rlo, rhi, sink, C);
      else filter_tile_q<CPL, true, 1>(pt, buf, cw0, lane, qc, edge, rlo, rhi, sink, C);
      break;
    case 2:
      if (wa) filter_tile_q<CPL, true, 2, Sink, true>(pt, buf, cw0, lane, qc, edge, rlo, rhi, sink, C);
      else filter_tile_q<CPL, true, 2>(pt, buf, cw0, lane, qc, edge, rlo, rhi, sink, C);
      break;
    default:
      if (wa) filter_tile_q<CPL, true, 3, Sink, true>(pt, buf, cw0, lane, qc, edge, rlo, rhi, sink, C);
      else filter_tile_q<CPL, true, 3>(pt, buf, cw0, lane, qc, edge, rlo, rhi, sink, C);
      break;
  }
}

// One BLOCK step (pattern offset off, broadcast symbol bc) over the CPL chunks of a lane.
template <int CPL, int Q>
__device__ __forceinline__ void block_step_q(Found4 (&F)[CPL], const uint8_t* cbase, uint32_t off, uint32_t bc,
                                             uint32_t k1) {
  const uint32_t sh = (off & 3u) * 8u;
  const uint8_t* b = cbase + (off & ~15u);
#pragma unroll
  for (int it = 0; it < CPL; ++it) found_and_eq(F[it], window16_q<Q>(b + it * 512u, sh), bc, k1);
}

template <int CPL>
__device__ __forceinline__ void block_step(Found4 (&F)[CPL], const uint8_t* cbase, uint32_t e) {
  const uint32_t off = e & 0xFFFFu, bc = (e >> 16) * 0x01010101u;
  const uint32_t k1 = 1u + (e >> 31);  // 1 (symbols < 256), opaque (eq_flags_fma)
  if ((off & 15u) == 0) {  // 16-B aligned window: one LDS.128, no shifts
#pragma unroll
    for (int it = 0; it < CPL; ++it) found_and_eq(F[it], lds128(cbase + off + it * 512u), bc, k1);
    return;
  }
  switch ((off >> 2) & 3u) {  // warp-uniform
    case 0: block_step_q<CPL, 0>(F, cbase, off, bc, k1); break;
    case 1: block_step_q<CPL, 1>(F, cbase, off, bc, k1); break;
    case 2: block_step_q<CPL, 2>(F, cbase, off, bc, k1); break;
    default: block_step_q<CPL, 3>(F, cbase, off, bc, k1); break;
  }
}

// One warp's share of a BLOCK tile: Alg. 4 on 16 alignments per lane-chunk.
template <int CPL>
__device__ __forceinline__ void block_tile(const Pat& pt, const uint8_t* buf, uint32_t cw0, int lane, bool edge,
                                           int32_t rlo, int32_t rhi, uint32_t* g_out, Ctr& C) {
  Found4 F[CPL];
#pragma unroll
  for (int it = 0; it < CPL; ++it)
    F[it] = edge ? found_from_mask16(range_mask16_rel((int32_t)(16u * (cw0 + it * 32u + lane)), rlo, rhi))
                 : found_all();
  const uint8_t* cbase = buf + 16u * (cw0 + lane);  // chunk it of this lane is at cbase + 512 * it
  uint32_t k = 0;
  // every window of a step lies inside the stage: 16c + (off & ~15) + 32 <= stage_len
#define SMGPU_BLOCK_DCHECK(e) \
  SMGPU_DCHECK(16u * (cw0 + (CPL - 1) * 32u + lane) + (((e) & 0xFFFFu) & ~15u) + 32u <= pt.lim)
  for (; k < pt.r; ++k) {  // peeled: all r, no test
    SMGPU_BLOCK_DCHECK(pt.tbl[k]);
    block_step<CPL>(F, cbase, pt.tbl[k]);
  }
  for (; k < pt.m; ++k) {  // ordered loop with exit test, warp-uniform
    uint32_t any = 0;
#pragma unroll
    for (int it = 0; it < CPL; ++it) any |= found_any(F[it]);
    if (!__any_sync(0xFFFFFFFFu, any != 0)) break;
    SMGPU_BLOCK_DCHECK(pt.tbl[k]);
    block_step<CPL>(F, cbase, pt.tbl[k]);
  }
#undef SMGPU_BLOCK_DCHECK
  if (!edge || (rlo < (int32_t)(16u * cw0 + 512u * CPL) && rhi > (int32_t)(16u * cw0))) {  // a valid warp-block
    C.add(kCtrBlocks, 1);
    C.add(kCtrSteps, k);
  }
#pragma unroll
  for (int it = 0; it < CPL; ++it) g_out[it] = compress_found(F[it]);  // popcount of found
}

// ---------------------------------------------------------------------------
// PACKED strategy (small text alphabets): every text byte is first replaced by a
// b-bit code, code(x) = (x >> s) & (2^b - 1), injective on the symbols of t (the
// host checks it on the histogram), and the packed codes of a tile are kept in
// shared memory.  A comparison step (Alg. 4) for pattern
// position pi(k) over 16 alignments is then a funnel shift of two code words, an
// XNOR with the broadcast code and an AND -- the SIMDcompare of PAPER.md:94 on
// b-bit lanes instead of 8-bit ones.  Same result as comparing bytes.
// ---------------------------------------------------------------------------
template <int B>
__device__ __forceinline__ uint32_t pack4(uint32_t w, uint32_t s) {
  if (B == 2) return (((w >> s) & 0x03030303u) * 0x01041040u) >> 24;  // byte k's code -> bits 2k, 2k+1
  return (((w >> s) & 0x01010101u) * 0x01020408u) >> 24;                 // byte k's code -> bit k
}
template <int B>
__device__ __forceinline__ uint32_t pack_chunk(const uint4 v, uint32_t s) {
  return pack4<B>(v.x, s) | (pack4<B>(v.y, s) << (4 * B)) | (pack4<B>(v.z, s) << (8 * B)) |
         (pack4<B>(v.w, s) << (12 * B));
}
template <int B>
__device__ __forceinline__ void store_codes(uint8_t* pk, uint32_t c, uint32_t codes) {
  if (B == 2) reinterpret_cast<uint32_t*>(pk)[c] = codes;
  else reinterpret_cast<uint16_t*>(pk)[c] = (uint16_t)codes;
}
// bit j -> bit 2j (16 -> 32 bits)
__device__ __forceinline__ uint32_t spread2(uint32_t x) {
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  return (x | (x << 1)) & 0x55555555u;
}
// bit 2j -> bit j
__device__ __forceinline__ uint32_t gather2(uint32_t x) {
  x &= 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0F0F0F0Fu;
  x = (x | (x >> 4)) & 0x00FF00FFu;
  return (x | (x >> 8)) & 0x0000FFFFu;
}

// One PACKED comparison step over the CPL chunks of a lane: F[it] &= [code of
// position 16c + off + j == ccode] for j = 0..15 (flag of alignment j at bit j for
// b = 1, bit 2j for b = 2).  W0/W1 = the code words holding positions 16c.. (kept in
// registers, so steps with off < 16 need no shared-memory load).  All branches
// are warp-uniform and taken once per step.
// MODE 0: branch on the window (warp-uniform); 1: register window known (off < 16);
// 2: shared-memory window known (off >= 16).
template <int CPL, int B, int MODE = 0>
__device__ __forceinline__ void packed_step(uint32_t (&F)[CPL], const uint32_t (&W0)[CPL], const uint32_t (&W1)[CPL],
                                            const uint32_t* pk32, uint32_t qbase, int lane, uint32_t e,
                                            uint32_t pk_words) {
  const uint32_t off = e & 0xFFFFu, ccode = e >> 16;
  const uint32_t rep = B == 2 ? ccode * 0x55555555u : 0u - ccode;
  // bit offset of position 16c + off relative to the start of W0 (lane parity matters for b = 1)
  const uint32_t u = B == 2 ? 2u * off : 16u * (uint32_t)(lane & 1) + off;
  if (MODE == 1 || (MODE == 0 && off < 16u)) {  // warp-uniform; then u < 32 on every lane
#pragma unroll
    for (int it = 0; it < CPL; ++it) {
      const uint32_t w = __funnelshift_r(W0[it], W1[it], u);
      if (B == 2) {
        const uint32_t x = ~(w ^ rep);
        F[it] &= x & (x >> 1);
      } else {
        F[it] &= ~(w ^ rep);
      }
    }
  } else {
    const uint32_t* p = pk32 + qbase + (u >> 5);  // word of chunk it at p[it * (B == 2 ? 32 : 16)]
    const uint32_t sh = u & 31u;
#pragma unroll
    for (int it = 0; it < CPL; ++it) {
      const uint32_t* pw = p + it * (B == 2 ? 32 : 16);
      SMGPU_DCHECK((uint32_t)(pw - pk32) + 1u < pk_words);
      const uint32_t w = __funnelshift_r(pw[0], pw[1], sh);
      if (B == 2) {
        const uint32_t x = ~(w ^ rep);
        F[it] &= x & (x >> 1);
      } else {
        F[it] &= ~(w ^ rep);
      }
    }
  }
}

// One warp's share of a PACKED tile: pack this lane's chunks (and a share of the
// halo), then -- after the CTA's consumer warps have packed the whole tile --
// Alg. 4 on the codes: r peeled steps, then the pi-ordered loop with a warp-uniform
// exit test.  Returns per-chunk 16-bit match masks.
// Returns the number of result units; unit i: mask m_out[i] (bit b <-> tile-relative
// alignment base_out[i] + b), units in ascending order within each lane-round.
// PRE (kPackedBPre): the stage already holds the tile's codes (packed once per call), so
// there is no packing, no CTA barrier, and the stage is released by the caller.
template <int CPL, int B, bool PRE = false>
__device__ __forceinline__ int packed_tile(const Pat& pt, const uint8_t* buf, uint8_t* pk, uint32_t pk_words,
                                           uint32_t nchunks,
                                            uint32_t code_shift, uint32_t cw0, int warp, int lane, bool edge,
                                            int32_t rlo, int32_t rhi, uint64_t* empty_bar, uint32_t* m_out,
                                            uint32_t* base_out, Ctr& C) {
  const bool valid_block = !edge || (rlo < (int32_t)(16u * cw0 + 512u * CPL) && rhi > (int32_t)(16u * cw0));
  if constexpr (PRE) {
    pk = const_cast<uint8_t*>(buf);
  } else {
#pragma unroll
    for (int it = 0; it < CPL; ++it) {
      const uint32_t c = cw0 + it * 32u + lane;
      store_codes<B>(pk, c, pack_chunk<B>(lds128(buf + 16u * c), code_shift));
    }
    for (uint32_t c = (uint32_t)CPL * kLanesPerTilePass + warp * 32u + lane; c < nchunks; c += kLanesPerTilePass) {
      SMGPU_DCHECK(16u * c + 16u <= pt.lim && (c + 1u) * 2u * B <= 4u * pk_words);
      store_codes<B>(pk, c, pack_chunk<B>(lds128(buf + 16u * c), code_shift));  // halo chunks
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_bar);  // the stage's bytes are no longer needed
    named_bar_sync(1, kConsumerWarps * 32);  // all codes of the tile are in place
  }
  const uint32_t* pk32 = reinterpret_cast<const uint32_t*>(pk);
  if constexpr (B == 1 && CPL >= 2) {
    // 1-bit codes: a lane compares a whole code word = 32 consecutive alignments per
    // step (double chunk dc = 32 alignments; warp w owns dc in [w*16*CPL, (w+1)*16*CPL)).
    constexpr int D = CPL / 2;
    const uint32_t dc0 = (cw0 >> 1) + lane;  // double chunk of it = 0; it-th at dc0 + 32 it
    uint32_t F[D], W0[D], W1[D];
#pragma unroll
    for (int it = 0; it < D; ++it) {
      const uint32_t dc = dc0 + it * 32u;
      F[it] = edge ? (range_mask16_rel((int32_t)(32u * dc), rlo, rhi) |
                      (range_mask16_rel((int32_t)(32u * dc + 16u), rlo, rhi) << 16))
                   : 0xFFFFFFFFu;
      SMGPU_DCHECK(dc + 1u < pk_words);
      W0[it] = pk32[dc];
      W1[it] = pk32[dc + 1];
    }
    // table entry e = off | (1 - code) << 31 (host, build_launch): the mask word
    // nrep = ~(code broadcast) in one arithmetic shift, so a step is F &= window ^ nrep
    // (one LOP3); the funnel shift takes e itself (amount mod 32)
    auto step_reg = [&](uint32_t e) {  // the window lies in W0:W1 (off < 32)
      const uint32_t nrep = (uint32_t)((int32_t)e >> 31);
#pragma unroll
      for (int it = 0; it < D; ++it) F[it] &= __funnelshift_r(W0[it], W1[it], e) ^ nrep;
    };
    auto step_mem = [&](uint32_t e) {  // off >= 32: two code words from shared memory
      const uint32_t nrep = (uint32_t)((int32_t)e >> 31);
      const uint32_t* p = pk32 + dc0 + ((e & 0xFFFFu) >> 5);
#pragma unroll
      for (int it = 0; it < D; ++it) {
        SMGPU_DCHECK((uint32_t)(p + it * 32 - pk32) + 1u < pk_words);
        F[it] &= __funnelshift_r(p[it * 32], p[it * 32 + 1], e) ^ nrep;
      }
    };
    auto step = [&](uint32_t e) {
      if ((e & 0xFFFFu) < 32u) step_reg(e);  // warp-uniform
      else step_mem(e);
    };
    // peeled: all r run, so their order is free -- the host put the r1
    // register-window steps first, leaving two branch-free loops
    uint32_t k = 0;
    for (; k < pt.r1; ++k) step_reg(pt.tbl[k]);
    for (; k < pt.r; ++k) step_mem(pt.tbl[k]);
    for (; k < pt.m; ++k) {                // ordered loop with exit test
      uint32_t any = 0;
#pragma unroll
      for (int it = 0; it < D; ++it) any |= F[it];
      if (!__any_sync(0xFFFFFFFFu, any != 0)) break;
      step(pt.tbl[k]);
    }
    if (valid_block) {
      C.add(kCtrBlocks, 1);
      C.add(kCtrSteps, k);
    }
#pragma unroll
    for (int it = 0; it < D; ++it) {
      m_out[it] = F[it];
      base_out[it] = 32u * (dc0 + it * 32u);
    }
    return D;
  }
  const uint32_t qbase = B == 2 ? (cw0 + lane) : ((cw0 + lane) >> 1);  // code word of chunk it = 0
  uint32_t F[CPL], W0[CPL], W1[CPL];
#pragma unroll
  for (int it = 0; it < CPL; ++it) {
    const uint32_t vm = edge ? range_mask16_rel((int32_t)(16u * (cw0 + it * 32u + lane)), rlo, rhi) : 0xFFFFu;
    F[it] = B == 2 ? spread2(vm) : vm;
    const uint32_t q = qbase + it * (B == 2 ? 32 : 16);
    SMGPU_DCHECK(q + 1u < pk_words);
    W0[it] = pk32[q];
    W1[it] = pk32[q + 1];
  }
  uint32_t k = 0;  // peeled: register-window steps first (see above)
  for (; k < pt.r1; ++k) packed_step<CPL, B, 1>(F, W0, W1, pk32, qbase, lane, pt.tbl[k], pk_words);
  for (; k < pt.r; ++k) packed_step<CPL, B, 2>(F, W0, W1, pk32, qbase, lane, pt.tbl[k], pk_words);
  for (; k < pt.m; ++k) {  // ordered loop with exit test, warp-uniform
    uint32_t any = 0;
#pragma unroll
    for (int it = 0; it < CPL; ++it) any |= F[it];
    if (!__any_sync(0xFFFFFFFFu, any != 0)) break;
    packed_step<CPL, B>(F, W0, W1, pk32, qbase, lane, pt.tbl[k], pk_words);
  }
  if (valid_block) {
    C.add(kCtrBlocks, 1);
    C.add(kCtrSteps, k);
  }
#pragma unroll
  for (int it = 0; it < CPL; ++it) {
    m_out[it] = B == 2 ? gather2(F[it]) : (F[it] & 0xFFFFu);
    base_out[it] = 16u * (cw0 + it * 32u + lane);
  }
  return CPL;
}

// Reporting (overflow pass): publish this warp's match count of item w, wait for the
// CTA's other compare warps, return the warp's first output index (tile offset +
// earlier warps).
__device__ __forceinline__ uint64_t publish_and_offset(const LaunchArgs& a, uint32_t* s_wt, uint32_t par, int warp,
                                                       int lane, uint64_t w, uint32_t wtot) {
  if (lane == 0) s_wt[par * kConsumerWarps + warp] = wtot;
  named_bar_sync(1, kConsumerWarps * 32);
  uint64_t run = a.tile_offsets[w];  // w = item index (d.item_base + ti) here
  for (int wv = 0; wv < warp; ++wv) run += s_wt[par * kConsumerWarps + wv];
  return run;
}

// Coalesced write of a warp's buffered positions (lane i writes entries i, i+32, ...).
__device__ __forceinline__ void write_list(const LaunchArgs& a, const uint16_t* list, uint32_t cnt, uint64_t run,
                                           int64_t pbase, int lane) {
  for (uint32_t i = lane; i < cnt; i += 32) {
    const uint64_t idx = run + i;
    if (idx < a.cap) a.pos[idx] = (uint64_t)(pbase + (int64_t)list[i]);
  }
}

// Reporting for strategies whose per-chunk results are still in registers.
template <bool IN_G, int CPL>
__device__ __forceinline__ void write_masks(const LaunchArgs& a, uint32_t* s_wt, uint16_t* list, uint32_t par,
                                            int warp, int lane, uint64_t w, uint32_t cw0, int64_t pos_base,
                                            const uint32_t (&mk)[CPL]) {
  AppendSink<IN_G> as{list};
#pragma unroll
  for (int it = 0; it < CPL; ++it) as(cw0 + it * 32u + lane, mk[it], lane);
  const uint64_t run = publish_and_offset(a, s_wt, par, warp, lane, w, as.n);
  __syncwarp();
  if (as.n <= (uint32_t)kListCap) {
    write_list(a, list, as.n, run, pos_base, lane);
  } else {
    WriteSink<IN_G> ws{run, pos_base, a.pos, a.cap};
#pragma unroll
    for (int it = 0; it < CPL; ++it) ws(cw0 + it * 32u + lane, mk[it], lane);
  }
}

// Reporting for PACKED: result units (mask, base) still in registers.
template <int CPL>
__device__ __forceinline__ void write_units(const LaunchArgs& a, uint32_t* s_wt, uint16_t* list, uint32_t par,
                                            int warp, int lane, uint64_t w, int64_t pos_base, const uint32_t (&mk)[CPL],
                                            const uint32_t (&mbase)[CPL], int units) {
  AppendSink<false> as{list};
#pragma unroll
  for (int it = 0; it < CPL; ++it)
    if (it < units) as.add(mbase[it], mk[it], lane);
  const uint64_t run = publish_and_offset(a, s_wt, par, warp, lane, w, as.n);
  __syncwarp();
  if (as.n <= (uint32_t)kListCap) {
    write_list(a, list, as.n, run, pos_base, lane);
  } else {
    WriteSink<false> ws{run, pos_base, a.pos, a.cap};
#pragma unroll
    for (int it = 0; it < CPL; ++it)
      if (it < units) ws.add(mbase[it], mk[it], lane);
  }
}

// Reporting pass 1 (kEpiStage): a warp's matches of a tile as per-chunk 16-bit masks
// in its shared bitmap bm[i] (chunk cw0 + i, bit b <-> u = 16 (cw0 + i) + b); FILTER
// writes only the chunks with matches, so its bitmap is kept clean between tiles.
struct StageSink {
  uint16_t* bm;
  uint32_t cw0;
  uint32_t n = 0;  // this lane's matches
  __device__ __forceinline__ void operator()(uint32_t c, uint32_t g, int) {
    if (g) {
      bm[c - cw0] = (uint16_t)g_to_mask16(g);
      n += __popc(g);
    }
  }
};

// Per-warp staging allocator: the warp owns a chunk of the pool and bump-allocates its
// records from it, so a record costs no global round trip.  Lane 0's copy is used.
struct StageAlloc {
  unsigned long long next = 0, end = 0;  // 16-B units
  // offset of `units` 16-B units followed by room for a terminator header, or
  // ~0ull when the pool is exhausted
  __device__ __forceinline__ unsigned long long take(const LaunchArgs& a, uint32_t units) {
    if (next + units + 1 > end) {
      const unsigned long long c = atomicAdd(a.stage_used, (unsigned long long)kStageChunk);
      if (c >= a.stage_cap16) return ~0ull;
      next = c;
      end = c + kStageChunk < a.stage_cap16 ? c + kStageChunk : a.stage_cap16;
      if (next + units + 1 > end) {  // (cannot happen: the host hands out whole chunks only)
        reinterpret_cast<uint4*>(a.stage)[c] = make_uint4(0u, 0u, 0u, 0u);  // the chunk holds no record
        return ~0ull;
      }
    }
    const unsigned long long o = next;
    next += units;  // the terminator slot is reused by the next record
    return o;
  }
};

// Reporting pass 1, one warp with wcnt > 0 matches in work item `item`: post its count
// (wc; the per-pattern total is accumulated by the caller like a count), then write its record -- the ascending u16 list of
// tile-relative alignments when sparse, its bitmap when dense -- followed by a zero
// terminator header.  No other warp is waited for.  If the pool is exhausted the item
// is queued (once) for the overflow pass, which recomputes it from the text.
template <int CPL, bool CLEAN>
__device__ __forceinline__ void stage_warp(const LaunchArgs& a, uint16_t* bm, StageAlloc& al,
                                           int warp, int lane, uint64_t item, int64_t pos_base, uint32_t wcnt) {
  constexpr uint32_t kWspan = 512u * CPL;  // alignments per warp (32 lanes x CPL chunks x 16)
  constexpr uint32_t kLog2Cpl = CPL == 8 ? 3 : CPL == 4 ? 2 : CPL == 2 ? 1 : 0;
  const bool as_list = rec_is_list(wcnt, kWspan, a.list_max);
  const uint32_t dbytes = rec_data_bytes(wcnt, kWspan, as_list);
  unsigned long long o = 0;
  if (lane == 0) {
    a.wc[item * kConsumerWarps + warp] = (uint16_t)wcnt;  // (the pattern total: the caller's acc)
    o = al.take(a, 1u + dbytes / 16u);
    if (o == ~0ull && !(atomicOr(&a.ovf_bits[item >> 5], 1u << (item & 31)) & (1u << (item & 31))))
      a.ovf_items[atomicAdd(a.ovf_n, 1u)] = (uint32_t)item;
  }
  o = __shfl_sync(0xFFFFFFFFu, o, 0);
  if (o != ~0ull) {
    uint8_t* rec = a.stage + o * 16u;
    if (lane == 0) {
      uint4 h;
      h.x = (uint32_t)(uint64_t)pos_base;
      h.y = (uint32_t)((uint64_t)pos_base >> 32);
      h.z = (uint32_t)item;
      h.w = wcnt | ((uint32_t)warp << 16) | (kLog2Cpl << 24) | (as_list ? 0u : kRecBitmap);
      reinterpret_cast<uint4*>(rec)[0] = h;
      reinterpret_cast<uint4*>(rec + kRecHeader + dbytes)[0] = make_uint4(0u, 0u, 0u, 0u);  // terminator
    }
    if (as_list) {  // sparse: ascending u16 list (lane l owns chunks [l CPL, l CPL + CPL))
      uint16_t mk[CPL];
      uint32_t pc = 0;
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        mk[j] = bm[lane * CPL + j];
        pc += __popc((uint32_t)mk[j]);
      }
      __syncwarp();  // every lane holds its masks: the list is built in place over the bitmap
      const uint32_t incl = warp_incl_scan(pc, lane);
      uint32_t idx = incl - pc;
      const uint32_t u0 = (uint32_t)warp * kWspan + 16u * (uint32_t)lane * CPL;
      // the lane's CPL 16-bit masks as one bit string (bit 16 j + k <-> alignment u0 + 16 j + k),
      // extracted in one loop: the warp iterates max-over-lanes(popcount) times, not once
      // per (chunk with a match in any lane)
      static_assert(CPL <= 8, "list extraction holds at most 128 mask bits per lane");
      uint64_t lo = 0, hi = 0;
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        if (j < 4) lo |= (uint64_t)mk[j] << (16 * j);
        else hi |= (uint64_t)mk[j] << (16 * (j - 4));
      }
      while (lo | hi) {
        uint32_t b;
        if (lo) {
          b = (uint32_t)__ffsll((long long)lo) - 1u;
          lo &= lo - 1;
        } else {
          b = 64u + (uint32_t)__ffsll((long long)hi) - 1u;
          hi &= hi - 1;
        }
        bm[idx++] = (uint16_t)(u0 + b);
      }
      __syncwarp();
      const uint4* src = reinterpret_cast<const uint4*>(bm);  // coalesced 16-B copy of the list
      uint4* dst = reinterpret_cast<uint4*>(rec + kRecHeader);
      for (uint32_t i = lane; i < dbytes / 16u; i += 32) dst[i] = src[i];
    } else {  // dense: the bitmap (64 CPL bytes)
      const uint4* src = reinterpret_cast<const uint4*>(bm);
      uint4* dst = reinterpret_cast<uint4*>(rec + kRecHeader);
#pragma unroll
      for (uint32_t i = lane; i < 4u * CPL; i += 32) dst[i] = src[i];
    }
  }
  if (CLEAN) {  // FILTER's bitmap must be clean for the next tile
    __syncwarp();
    uint32_t* bw = reinterpret_cast<uint32_t*>(bm);
#pragma unroll
    for (uint32_t i = lane; i < 16u * CPL; i += 32) bw[i] = 0u;
  }
  __syncwarp();
}

}  // namespace

// NEXT-4 epilogue (kEpiCountMc launches): the last CTA to finish reads the
// launch's per-pattern counts (complete: every CTA's atomics happened before its
// done_ctr increment, fenced) and one warp adds each to the NVLink multicast address
// with multimem.red -- the all-reduce of PAPER.md:36's counting version across ranks,
// done by the switch, no collective call and no extra launch.  Only the kEpiCountMc
// instantiations contain it: inline asm is convergent, and its presence anywhere in a
// kernel made the compiler wrap the kernel's divergent regions in reconvergence
// barriers (PAIR count kernel: 84 -> 213 BSSY, about -4 % on every count launch).
template <int CAP>
__device__ __forceinline__ void nvls_epilogue(const LaunchParams<CAP>& P, int warp, int lane, uint32_t* s_flag) {
  const LaunchArgs& a = P.a;
  named_bar_sync(1, kConsumerWarps * 32);  // this CTA's compare warps have all added their counts
  if (warp == 0 && lane == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(a.done_ctr, 1u);
    s_flag[0] = prev == gridDim.x - 1 ? 1u : 0u;
  }
  named_bar_sync(1, kConsumerWarps * 32);
  if (s_flag[0] == 0u || warp != 0) return;
  __threadfence();  // the other CTAs' count atomics are visible
  for (uint32_t i = lane; i < a.npat; i += 32) {
    uint64_t* local = P.d[i].count_out;
    const unsigned long long v = *reinterpret_cast<volatile unsigned long long*>(local);
    uint64_t* mc = a.mc_base + (local - a.local_base);
    if (!v) continue;
    if (a.mc_emulate) atomicAdd(reinterpret_cast<unsigned long long*>(mc), v);
    else multimem_red_add_u64(mc, v);
  }
}

// ---------------------------------------------------------------------------
// the kernel: a batch of patterns, each a full pass over the text; work item w
// = (pattern k, tile ti) in pattern-major order, round-robin over persistent CTAs
// (one CTA flows from one pattern's last tiles into the next pattern's first).
// ---------------------------------------------------------------------------
// 3 CTAs per SM (2-stage rings of 32 KiB tiles): FILTER, PAIR and PACKED-PRE are
// register-capped for 3 (BLOCK's Found4[CPL] registers would spill; per-tile PACKED is
// held to 2 CTAs by its code buffers anyway; the overflow pass is rarely active)
template <int STRAT, int EPI, int CAP, int CPL>
__global__ void __launch_bounds__(kThreads,
                                  ((STRAT == kFilter || STRAT == kPair || is_prepacked(STRAT)) && EPI != kEpiWrite)
                                      ? 3
                                      : 2)
    search_kernel(const __grid_constant__ LaunchParams<CAP> P) {
  extern __shared__ __align__(128) uint8_t smem[];
  const LaunchArgs& a = P.a;
  if (a.guard_mode) {  // PACKED on a caller histogram, or its fallback: exactly one of the pair runs
    const uint32_t g = *reinterpret_cast<const volatile uint32_t*>(a.guard);
    if ((g != 0u) != (a.guard_mode == kGuardSet)) return;
  }
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  uint32_t* s_wt = reinterpret_cast<uint32_t*>(smem + kWarpTotOff);  // [2][W]
  uint4* tix = reinterpret_cast<uint4*>(smem + kTixOff);             // [stages] dispatched items
  uint8_t* ring = smem + a.ring_off;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    if (lane == 0) produce<EPI, CAP, is_prepacked(STRAT), code_bits(STRAT)>(P, ring, full, empty, tix);
    return;
  }

  uint16_t* qc = reinterpret_cast<uint16_t*>(smem + kQueueOff) + warp * kQueueLen;
  // reporting only: kEpiWrite position list (kListCap u16) / kEpiStage bitmap (32 CPL u16)
  uint16_t* list = reinterpret_cast<uint16_t*>(smem + a.list_off) + warp * (EPI == kEpiWrite ? kListCap : 32 * CPL);
  StageAlloc salloc;     // kEpiStage: this warp's staging-pool chunk
  if (EPI == kEpiStage) {  // the bitmap starts clean
    uint32_t* bw = reinterpret_cast<uint32_t*>(list);
    for (uint32_t i = lane; i < 16u * CPL; i += 32) bw[i] = 0u;
    __syncwarp();
  }
  const uint32_t T = a.tile;
  const uint32_t cw0 = (uint32_t)warp * 32u * CPL;  // first chunk of this warp
  uint32_t s = 0, ph = 0, par = 0, par_pk = 0;
  uint32_t kc = 0;   // count / stage: pattern whose matches `acc` holds
  uint32_t acc = 0;  // count / stage: this lane's matches of pattern kc so far
  Ctr C;
#ifdef SMGPU_COUNTERS
  C.v[kCtrAlphaEff] = (STRAT == kFilter || STRAT == kPair) ? 0ull : 512ull * CPL;
#endif
  WorkIter<EPI, CAP> items(P);
  const bool dyn = EPI != kEpiWrite && a.work_ctr != nullptr;
  uint32_t k;
  uint64_t ti;
  bool pub_edge = false;
  while (true) {
    if (dyn) {  // the stage's item, published by the producer with the stage
      if (a.wait_ns) mbar_wait_sleep(&full[s], ph, a.wait_ns);
      else mbar_wait(&full[s], ph);
      const uint4 tw = tix[s];  // {w, k, ti, edge}, mapped by the producer
      if (tw.x == kNoItem) break;
      k = tw.y;
      ti = tw.z;
      pub_edge = tw.w != 0u;
    } else if (!items.advance(P, k, ti)) {
      break;
    }
    C.add(kCtrWarpTiles, 1);
    if (EPI != kEpiWrite && k != kc) {  // flush pattern kc (warp-uniform; k only grows here)
      const uint32_t ws = __reduce_add_sync(0xFFFFFFFFu, acc);
      if (lane == 0 && ws) count_add(a, P.d[kc].count_out, ws);
      acc = 0;
      kc = k;
    }
    const PatDesc& d = P.d[k];
    const uint64_t item = d.item_base + ti;
    if (!dyn) {
      if (a.wait_ns) mbar_wait_sleep(&full[s], ph, a.wait_ns);
      else mbar_wait(&full[s], ph);
    }
    const uint8_t* buf = ring + (size_t)s * a.stage_stride;
    const Pat pt{d.m, d.r, d.a1, d.bc1, d.s2, d.bc2, d.pre, (d.flags >> 8) & 0xFFu, d.stage_len, P.e + d.tbl};
    const bool edge = dyn ? pub_edge : (ti < d.edge_lo || ti >= d.edge_hi);  // tile holds invalid alignments
    const int64_t shift = (STRAT == kFilter || STRAT == kPair) ? (int64_t)d.a1 : 0;
    const int64_t x_base = (int64_t)((d.k_begin + ti) * T) - shift;  // alignment offset of u = 0
    const int64_t pos_base = x_base - (int64_t)a.delta + (int64_t)a.pos_offset;  // position of u = 0
    int32_t rlo = 0, rhi = (int32_t)T;
    if (edge) {
      const int64_t vlo = (int64_t)a.delta, vhi = (int64_t)(a.delta + d.A);
      rlo = (int32_t)imin(imax(vlo - x_base, 0), (int64_t)T);
      rhi = (int32_t)imin(imax(vhi - x_base, 0), (int64_t)T);
    }
    bool released = false;  // the stage's bytes were handed back to the producer

    if (STRAT == kFilter || STRAT == kPair) {
      auto ftile = [&](auto& sink, Ctr& cc) {
        if constexpr (STRAT == kPair) pair_tile<CPL>(pt, buf, cw0, lane, qc, edge, rlo, rhi, sink, cc);
        else filter_tile<CPL>(pt, buf, cw0, lane, qc, edge, rlo, rhi, sink, cc);
      };
      if (is_count_epi(EPI)) {
        CountSink cs;
        ftile(cs, C);
        acc += cs.n;
      } else if (EPI == kEpiStage) {
        StageSink sk{list, cw0};
        ftile(sk, C);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        released = true;
        acc += sk.n;
        const uint32_t wcnt = __reduce_add_sync(0xFFFFFFFFu, sk.n);
        if (wcnt) stage_warp<CPL, true>(a, list, salloc, warp, lane, item, pos_base, wcnt);
      } else {  // overflow pass: buffer this warp's matches, exchange warp totals, write coalesced
        AppendSink<true> as{list};
        ftile(as, C);
        uint64_t run = publish_and_offset(a, s_wt, par, warp, lane, item, as.n);
        if (as.n <= (uint32_t)kListCap) {
          write_list(a, list, as.n, run, pos_base, lane);
        } else {  // list overflow (very dense tile): ranked writes from a recomputation
          WriteSink<> ws{run, pos_base, a.pos, a.cap};
          {
            Ctr C2;  // a recomputation: not counted again
            ftile(ws, C2);
          }
        }
        par ^= 1u;
      }
    } else if (is_packed(STRAT)) {
      constexpr int B = code_bits(STRAT);
      constexpr bool PRE = is_prepacked(STRAT);
      uint32_t mk[CPL], mbase[CPL];
      uint8_t* pk = smem + a.pack_off + par_pk * a.pack_bytes;
      const int units = packed_tile<CPL, B, PRE>(pt, buf, pk, PRE ? d.stage_len / 4u : a.pack_bytes / 4u,
                                                 d.stage_len / 16u, a.code_shift, cw0, warp, lane, edge, rlo, rhi,
                                                 &empty[s], mk, mbase, C);
      released = !PRE;  // packed_tile released the stage after packing (PRE: it was read until now)
      par_pk ^= 1u;
      uint32_t tc = 0;
#pragma unroll
      for (int it = 0; it < CPL; ++it)
        if (it < units) tc += __popc(mk[it]);
      if (is_count_epi(EPI)) {
        acc += tc;
      } else if (EPI == kEpiStage) {
        constexpr bool kWide = B == 1 && CPL >= 2;  // 32-bit masks of 32 alignments
        acc += tc;
        const uint32_t wcnt = __reduce_add_sync(0xFFFFFFFFu, tc);
        if (wcnt) {
#pragma unroll
          for (int it = 0; it < CPL; ++it) {
            if (it >= units) break;
            const uint32_t rel = mbase[it] / 16u - cw0;  // chunk index within the warp
            if (kWide) reinterpret_cast<uint32_t*>(list)[rel / 2u] = mk[it];
            else list[rel] = (uint16_t)mk[it];
          }
          __syncwarp();
          stage_warp<CPL, false>(a, list, salloc, warp, lane, item, pos_base, wcnt);
        }
      } else {
        write_units<CPL>(a, s_wt, list, par, warp, lane, item, pos_base, mk, mbase, units);
        par ^= 1u;
      }
    } else {
      uint32_t g[CPL];
      block_tile<CPL>(pt, buf, cw0, lane, edge, rlo, rhi, g, C);
      uint32_t tc = 0;
#pragma unroll
      for (int it = 0; it < CPL; ++it) tc += __popc(g[it]);
      if (is_count_epi(EPI)) {
        acc += tc;
      } else if (EPI == kEpiStage) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        released = true;
        acc += tc;
        const uint32_t wcnt = __reduce_add_sync(0xFFFFFFFFu, tc);
        if (wcnt) {
#pragma unroll
          for (int it = 0; it < CPL; ++it) list[it * 32 + lane] = (uint16_t)g_to_mask16(g[it]);
          __syncwarp();
          stage_warp<CPL, false>(a, list, salloc, warp, lane, item, pos_base, wcnt);
        }
      } else {
        write_masks<true, CPL>(a, s_wt, list, par, warp, lane, item, cw0, pos_base, g);
        par ^= 1u;
      }
    }

    __syncwarp();
    if (!released && lane == 0) mbar_arrive(&empty[s]);
    if (++s == a.stages) {
      s = 0;
      ph ^= 1u;
    }
  }

  if (EPI != kEpiWrite) {
    const uint32_t ws = __reduce_add_sync(0xFFFFFFFFu, acc);
    if (lane == 0 && ws) count_add(a, P.d[kc].count_out, ws);
  }
  C.flush(a.ctr, lane);
  if constexpr (EPI == kEpiCountMc) nvls_epilogue(P, warp, lane, s_wt);
}

}  // namespace smgpu
