// search_kernel.cu -- the hot path: exact occurrence counting / reporting of a
// pattern in a device-resident byte text, pattern symbols compared rarest-first
// with peeled first comparisons (Algs. 3-4), B200-native.
//
// One persistent CTA per SM: warp 8 is the TMA producer, warps 0..7 compare.
//   * A3 staging (PAPER.md:101-106 loads 16/32 unaligned bytes; here): tiles of
//     T text bytes plus the pattern's halo are copied HBM -> shared memory with
//     1-D TMA bulk copies (cp.async.bulk, 16-B granules, L2 evict-first) into a
//     ring of mbarrier-guarded stages.  Ragged 16-B ends of the text are loaded
//     byte-wise by the producer so nothing outside t[0..n) is read.
//   * The SIMDcompare primitive becomes a packed-byte compare:
//     each lane owns chunks of 16 consecutive alignments held as 4 x u32 words
//     with one flag bit (0x80) per alignment.
//   * FILTER strategy: the first comparison pi(1) -- the rarest symbol, where the
//     paper's frequency order pays most -- runs over the chunk
//     with aligned 16-B shared loads; each surviving alignment continues with
//     pi(2..m) and early exit (Alg. 3's inner loop at alpha = 1).
//   * BLOCK strategy: Alg. 4: r peeled comparisons without a
//     test, then the pi-ordered loop with a warp-uniform exit
//     test (__any_sync) over all alignments the warp holds.
//   * A6: popcount -> warp reduce -> one u64 atomic per warp.
//   * A8: reporting writes ascending positions from a per-tile exclusive prefix.
#include "device_util.cuh"
#include "launch.h"
#include "search.cuh"

namespace smgpu {

namespace {

__device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

// bits b in [0,16) with lo <= x0 + b < hi
__device__ __forceinline__ uint32_t range_mask16(int64_t x0, int64_t lo, int64_t hi) {
  int64_t l = lo - x0, h = hi - x0;
  l = imin(imax(l, 0), 16);
  h = imin(imax(h, 0), 16);
  if (h <= l) return 0u;
  return ((1u << (uint32_t)h) - 1u) & ~((1u << (uint32_t)l) - 1u);
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------
// TMA producer (one thread)
// ---------------------------------------------------------------------------
template <int EPI>
__device__ void produce(const SearchArgs& a, uint8_t* ring, uint64_t* full, uint64_t* empty) {
  const uint64_t pol = l2_policy_evict_first();
  const int64_t tlo = (int64_t)a.delta, thi = (int64_t)(a.delta + a.n);
  uint32_t j = 0;
  for (uint64_t ti = blockIdx.x; ti < a.ntiles; ti += gridDim.x) {
    if (EPI == kEpiWrite && a.tile_offsets[ti + 1] == a.tile_offsets[ti]) continue;
    const uint32_t s = j % a.stages;
    const uint32_t u = j / a.stages;
    if (u > 0) mbar_wait(&empty[s], (u & 1u) ^ 1u);
    uint8_t* buf = ring + (size_t)s * a.stage_stride;
    const int64_t lo = (int64_t)((a.k_begin + ti) * a.tile) - (int64_t)a.pre;
    const int64_t hi = lo + (int64_t)a.stage_len;
    const int64_t vlo = imax(lo, tlo), vhi = imin(hi, thi);
    uint32_t tx = 0;
    int64_t alo = 0;
    if (vlo < vhi) {
      alo = (vlo + 15) & ~(int64_t)15;
      const int64_t ahi = vhi & ~(int64_t)15;
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
    if (tx) tma_load_1d(buf + (alo - lo), a.base + alo, tx, &full[s], pol);
    ++j;
  }
}

// ---------------------------------------------------------------------------
// FILTER strategy: one chunk of 16 alignments whose pi(1)-bytes are the 16
// aligned bytes v (y-space: byte y <-> alignment y - a1).  Returns the 16-bit
// match mask (bit b <-> alignment x0 + b) of the chunk's valid alignments.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t filter_verify(const uint4 v, uint32_t bc1, const uint8_t* xbuf,
                                                  uint32_t vmask, const uint32_t* tbl, uint32_t m) {
  uint32_t mk = flags_to_nibble(eq_flags(v.x, bc1)) | (flags_to_nibble(eq_flags(v.y, bc1)) << 4) |
                (flags_to_nibble(eq_flags(v.z, bc1)) << 8) | (flags_to_nibble(eq_flags(v.w, bc1)) << 12);
  mk &= vmask;
  uint32_t out = 0;
  while (mk) {
    const uint32_t b = __ffs(mk) - 1;
    mk &= mk - 1;
    const uint8_t* xp = xbuf + b;  // shared-memory address of alignment x0 + b
    uint32_t q = 1;
    for (; q < m; ++q) {  // pi(2..m), early exit on the first mismatch (Alg. 3 inner loop)
      const uint32_t e = tbl[q];
      if (xp[e & 0xFFFFu] != (e >> 16)) break;
    }
    if (q == m) out |= 1u << b;
  }
  return out;
}

// ---------------------------------------------------------------------------
// BLOCK strategy helpers
// ---------------------------------------------------------------------------
struct Found4 {
  uint32_t f0, f1, f2, f3;
};

// found &= SIMDcompare(t, x + off, p, pi(q)) for 16 alignments of one lane-chunk
__device__ __forceinline__ void block_step(Found4& F, const uint8_t* cbuf, uint32_t off, uint32_t bc) {
  const uint8_t* src = cbuf + (off & ~15u);
  const uint4 lo = lds128(src);
  const uint4 hi = lds128(src + 16);
  const uint32_t sh = (off & 3u) * 8u;
  uint32_t w0, w1, w2, w3;
  switch ((off >> 2) & 3u) {
    case 0:
      w0 = byte_window(lo.x, lo.y, sh); w1 = byte_window(lo.y, lo.z, sh);
      w2 = byte_window(lo.z, lo.w, sh); w3 = byte_window(lo.w, hi.x, sh);
      break;
    case 1:
      w0 = byte_window(lo.y, lo.z, sh); w1 = byte_window(lo.z, lo.w, sh);
      w2 = byte_window(lo.w, hi.x, sh); w3 = byte_window(hi.x, hi.y, sh);
      break;
    case 2:
      w0 = byte_window(lo.z, lo.w, sh); w1 = byte_window(lo.w, hi.x, sh);
      w2 = byte_window(hi.x, hi.y, sh); w3 = byte_window(hi.y, hi.z, sh);
      break;
    default:
      w0 = byte_window(lo.w, hi.x, sh); w1 = byte_window(hi.x, hi.y, sh);
      w2 = byte_window(hi.y, hi.z, sh); w3 = byte_window(hi.z, hi.w, sh);
      break;
  }
  F.f0 &= eq_flags_raw(w0, bc);
  F.f1 &= eq_flags_raw(w1, bc);
  F.f2 &= eq_flags_raw(w2, bc);
  F.f3 &= eq_flags_raw(w3, bc);
}

__device__ __forceinline__ Found4 found_init(uint32_t vmask) {
  if (vmask == 0xFFFFu) return Found4{0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u};
  return Found4{nibble_to_flags(vmask & 0xFu), nibble_to_flags((vmask >> 4) & 0xFu),
                nibble_to_flags((vmask >> 8) & 0xFu), nibble_to_flags((vmask >> 12) & 0xFu)};
}

__device__ __forceinline__ uint32_t found_mask16(const Found4& F) {
  return flags_to_nibble(F.f0) | (flags_to_nibble(F.f1) << 4) | (flags_to_nibble(F.f2) << 8) |
         (flags_to_nibble(F.f3) << 12);
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t u = __shfl_up_sync(0xFFFFFFFFu, v, d);
    if (lane >= d) v += u;
  }
  return v;
}

}  // namespace

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <int STRAT, int EPI, int MAXM, int CPL>
__global__ void __launch_bounds__(kThreads, 1) search_kernel(const SearchArgs a, const PatternTable<MAXM> pt) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  uint32_t* s_wt = reinterpret_cast<uint32_t*>(smem + 2 * kMaxStages * sizeof(uint64_t));  // [2][CPL][W]
  uint32_t* tbl = reinterpret_cast<uint32_t*>(smem + a.tbl_off);
  uint8_t* ring = smem + a.ring_off;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t q = threadIdx.x; q < a.m; q += blockDim.x) tbl[q] = pt.e[q];
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    if (lane == 0) produce<EPI>(a, ring, full, empty);
    return;
  }

  const uint32_t m = a.m, T = a.tile;
  const int64_t tlo = (int64_t)a.delta, thi = (int64_t)(a.delta + a.A);  // valid alignment offsets
  uint32_t cnt = 0;
  uint32_t j = 0, par = 0;
  for (uint64_t ti = blockIdx.x; ti < a.ntiles; ti += gridDim.x) {
    if (EPI == kEpiWrite && a.tile_offsets[ti + 1] == a.tile_offsets[ti]) continue;
    const uint32_t s = j % a.stages;
    mbar_wait(&full[s], (j / a.stages) & 1u);
    const uint8_t* buf = ring + (size_t)s * a.stage_stride;
    const int64_t kT = (int64_t)((a.k_begin + ti) * T);

    uint32_t res[CPL];
    int64_t x0[CPL];  // alignment offset of bit 0 of each chunk
    if (STRAT == kFilter) {
      const int64_t xlo = imax(tlo, kT - (int64_t)a.a1), xhi = imin(thi, kT + (int64_t)T - (int64_t)a.a1);
      uint4 v[CPL];
#pragma unroll
      for (int it = 0; it < CPL; ++it) {
        const uint32_t c = it * kLanesPerTilePass + warp * 32 + lane;
        v[it] = lds128(buf + a.pre + 16u * c);
        x0[it] = kT + 16 * (int64_t)c - (int64_t)a.a1;
      }
#pragma unroll
      for (int it = 0; it < CPL; ++it) {
        const uint32_t z = (any_eq_term(v[it].x, a.bc1) | any_eq_term(v[it].y, a.bc1) |
                            any_eq_term(v[it].z, a.bc1) | any_eq_term(v[it].w, a.bc1)) &
                           0x80808080u;
        res[it] = 0;
        if (z) {
          const uint32_t c = it * kLanesPerTilePass + warp * 32 + lane;
          const uint32_t vm = range_mask16(x0[it], xlo, xhi);
          res[it] = filter_verify(v[it], a.bc1, buf + a.pre + 16u * c - a.a1, vm, tbl, m);
        }
      }
    } else {
      const int64_t xlo = imax(tlo, kT), xhi = imin(thi, kT + (int64_t)T);
      Found4 F[CPL];
#pragma unroll
      for (int it = 0; it < CPL; ++it) {
        const uint32_t c = it * kLanesPerTilePass + warp * 32 + lane;
        x0[it] = kT + 16 * (int64_t)c;
        F[it] = found_init(range_mask16(x0[it], xlo, xhi));
      }
      uint32_t q = 0;
      for (; q < a.r; ++q) {  // peeled: all r comparisons, no test
        const uint32_t e = tbl[q];
        const uint32_t off = e & 0xFFFFu, bc = (e >> 16) * 0x01010101u;
#pragma unroll
        for (int it = 0; it < CPL; ++it)
          block_step(F[it], buf + 16u * (it * kLanesPerTilePass + warp * 32 + lane), off, bc);
      }
      for (; q < m; ++q) {  // ordered loop with exit test, warp-uniform
        uint32_t any = 0;
#pragma unroll
        for (int it = 0; it < CPL; ++it) any |= F[it].f0 | F[it].f1 | F[it].f2 | F[it].f3;
        if (!__any_sync(0xFFFFFFFFu, (any & 0x80808080u) != 0)) break;
        const uint32_t e = tbl[q];
        const uint32_t off = e & 0xFFFFu, bc = (e >> 16) * 0x01010101u;
#pragma unroll
        for (int it = 0; it < CPL; ++it)
          block_step(F[it], buf + 16u * (it * kLanesPerTilePass + warp * 32 + lane), off, bc);
      }
#pragma unroll
      for (int it = 0; it < CPL; ++it) {
        F[it].f0 &= 0x80808080u; F[it].f1 &= 0x80808080u; F[it].f2 &= 0x80808080u; F[it].f3 &= 0x80808080u;
        res[it] = (EPI == kEpiWrite) ? found_mask16(F[it])
                                     : (uint32_t)__popc(F[it].f0 | (F[it].f1 >> 1) | (F[it].f2 >> 2) | (F[it].f3 >> 3));
      }
    }

    if (EPI == kEpiCount || EPI == kEpiTileCount) {
      uint32_t tc = 0;
#pragma unroll
      for (int it = 0; it < CPL; ++it) tc += (STRAT == kFilter) ? (uint32_t)__popc(res[it]) : res[it];
      if (EPI == kEpiCount) {
        cnt += tc;
      } else {
        const uint32_t ws = __reduce_add_sync(0xFFFFFFFFu, tc);
        if (lane == 0 && ws) atomicAdd(reinterpret_cast<unsigned long long*>(&a.tile_counts[ti]),
                                       (unsigned long long)ws);
      }
    } else {  // kEpiWrite: ascending positions from the tile's exclusive prefix
      uint32_t c_it[CPL], incl[CPL];
#pragma unroll
      for (int it = 0; it < CPL; ++it) {
        c_it[it] = (uint32_t)__popc(res[it]);
        incl[it] = warp_incl_scan(c_it[it], lane);
        if (lane == 31) s_wt[(par * CPL + it) * kConsumerWarps + warp] = incl[it];
      }
      named_bar_sync(1, kConsumerWarps * 32);
      uint64_t run = a.tile_offsets[ti];
#pragma unroll
      for (int it = 0; it < CPL; ++it) {
        uint32_t before = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) {
          const uint32_t vv = s_wt[(par * CPL + it) * kConsumerWarps + w];
          tot += vv;
          before += (w < warp) ? vv : 0u;
        }
        uint64_t idx = run + before + incl[it] - c_it[it];
        uint32_t mk = res[it];
        while (mk) {
          const uint32_t b = __ffs(mk) - 1;
          mk &= mk - 1;
          if (idx < a.cap) a.pos[idx] = (uint64_t)(x0[it] + (int64_t)b - (int64_t)a.delta);
          ++idx;
        }
        run += tot;
      }
      par ^= 1u;
    }

    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    ++j;
  }

  if (EPI == kEpiCount) {
    const uint32_t ws = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if (lane == 0 && ws) atomicAdd(reinterpret_cast<unsigned long long*>(a.count_out), (unsigned long long)ws);
  }
}

// ---------------------------------------------------------------------------
// host-side dispatch over the template parameters
// ---------------------------------------------------------------------------
namespace {

template <int STRAT, int EPI, int MAXM, int CPL>
cudaError_t launch_one(const SearchArgs& a, const uint32_t* e, uint32_t m, int grid, size_t smem,
                       cudaStream_t st) {
  auto kfn = search_kernel<STRAT, EPI, MAXM, CPL>;
  static bool attr_done = false;  // benign race: idempotent attribute set
  if (!attr_done) {
    cudaError_t err = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (err != cudaSuccess) return err;
    attr_done = true;
  }
  PatternTable<MAXM> pt;
  for (uint32_t q = 0; q < m; ++q) pt.e[q] = e[q];
  for (uint32_t q = m; q < (uint32_t)MAXM; ++q) pt.e[q] = 0;
  kfn<<<grid, kThreads, smem, st>>>(a, pt);
  return cudaGetLastError();
}

template <int STRAT, int EPI, int CPL>
cudaError_t launch_m(const SearchArgs& a, const uint32_t* e, uint32_t m, int grid, size_t smem,
                     cudaStream_t st) {
  if (m <= 64) return launch_one<STRAT, EPI, 64, CPL>(a, e, m, grid, smem, st);
  if (m <= 1024) return launch_one<STRAT, EPI, 1024, CPL>(a, e, m, grid, smem, st);
  return launch_one<STRAT, EPI, 4096, CPL>(a, e, m, grid, smem, st);
}

template <int STRAT, int EPI>
cudaError_t launch_c(const SearchArgs& a, const uint32_t* e, uint32_t m, int cpl, int grid, size_t smem,
                     cudaStream_t st) {
  if (cpl == 4) return launch_m<STRAT, EPI, 4>(a, e, m, grid, smem, st);
  return launch_m<STRAT, EPI, 1>(a, e, m, grid, smem, st);
}

template <int STRAT>
cudaError_t launch_e(const SearchArgs& a, const uint32_t* e, uint32_t m, int epi, int cpl, int grid,
                     size_t smem, cudaStream_t st) {
  if (epi == kEpiCount) return launch_c<STRAT, kEpiCount>(a, e, m, cpl, grid, smem, st);
  if (epi == kEpiTileCount) return launch_c<STRAT, kEpiTileCount>(a, e, m, cpl, grid, smem, st);
  return launch_c<STRAT, kEpiWrite>(a, e, m, cpl, grid, smem, st);
}

}  // namespace

cudaError_t launch_search(const SearchArgs& a, const uint32_t* table, int strategy, int epilogue, int cpl,
                          int grid, size_t smem_bytes, cudaStream_t stream) {
  if (strategy == kFilter) return launch_e<kFilter>(a, table, a.m, epilogue, cpl, grid, smem_bytes, stream);
  return launch_e<kBlock>(a, table, a.m, epilogue, cpl, grid, smem_bytes, stream);
}

}  // namespace smgpu
