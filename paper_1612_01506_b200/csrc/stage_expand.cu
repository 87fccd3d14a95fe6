// stage_expand.cu -- reporting (A8, "printing position i"): turn the
// staged match records of reporting pass 1 (kEpiStage, search.cuh / search_impl.cuh)
// into ascending 0-based positions.  The matches of compare warp w in work item
// `item` go to pos[tile_offsets[item] + sum_{w' < w} wc[item][w'] ..): items in the
// scanned (pattern-major, tile-ascending) order, warps ascending within an item,
// alignments ascending within a warp -- the order of Alg. 1's loop.
// Only the staging pool is read, never the text.
//
// One warp per pool chunk (8 KiB): the chunk is pulled into shared memory with
// independent 16-B loads, lane 0 walks its record chain (up to the zero terminator),
// the lanes fetch the records' output offsets in parallel, then the u16 lists of all
// the chunk's records are written as one flattened sequence (32 consecutive elements
// per warp store), and bitmap records 32 x 32 alignments per round through a shared
// index buffer, so that the 8-byte position stores are coalesced.
#include "device_util.cuh"
#include "launch.h"

namespace smgpu {
namespace {

constexpr int kExpandWarps = 8;
constexpr uint32_t kChunkBytes = kStageChunk * 16u;
constexpr uint32_t kMaxRecs = kStageChunk / 2u;  // a record is >= 2 units (header + data)
// per warp: chunk | rout u64[kMaxRecs] | rpre u32[kMaxRecs + 1] | roff u16[kMaxRecs] | sbuf u16[1024]
constexpr uint32_t kWarpSmem = (kChunkBytes + kMaxRecs * 8u + (kMaxRecs + 1u) * 4u + kMaxRecs * 2u + 2048u + 15u) & ~15u;

__device__ __forceinline__ uint32_t warp_incl_scan_x(uint32_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, v, d);
    if (lane >= d) v += u;
  }
  return v;
}

__device__ __forceinline__ bool is_list_record(uint32_t hw) { return (hw & kRecBitmap) == 0u; }
__device__ __forceinline__ uint32_t rec_wspan(uint32_t hw) { return 512u << ((hw >> 24) & 3u); }

// a bitmap record: bit b of u32 word i <-> u = w wspan + 32 i + b
__device__ __forceinline__ void write_bitmap(const uint8_t* rec, uint64_t out, uint64_t* pos, uint64_t cap,
                                             uint16_t* sbuf, int lane) {
  const uint4 h = *reinterpret_cast<const uint4*>(rec);
  const int64_t pos_base = (int64_t)(((uint64_t)h.y << 32) | h.x);
  const uint32_t w = (h.w >> 16) & 0xFFu;
  const uint32_t wspan = rec_wspan(h.w);
  const uint8_t* data = rec + kRecHeader;
  const uint32_t* bm = reinterpret_cast<const uint32_t*>(data);
  const uint32_t words = wspan / 32u;
  uint64_t o = out;
  for (uint32_t r0 = 0; r0 < words && o < cap; r0 += 32) {
    const uint32_t i = r0 + lane;
    uint32_t mk = i < words ? bm[i] : 0u;
    if (r0 + 32 <= words && __all_sync(0xFFFFFFFFu, mk == 0xFFFFFFFFu)) {
      // every alignment of the round matches: 1024 consecutive positions, written with
      // 16-B stores (an odd head position first when pos + o is not 16-B aligned)
      const uint64_t b0 = (uint64_t)(pos_base + (int64_t)(w * wspan + 32u * r0));
      uint64_t* dst = pos + o;
      if (o + 1024u <= cap) {
        const uint32_t head = (uint32_t)((reinterpret_cast<uintptr_t>(dst) >> 3) & 1u);
        if (head && lane == 0) dst[0] = b0;
        ulonglong2* d2 = reinterpret_cast<ulonglong2*>(dst + head);
        const uint32_t npairs = (1024u - head) / 2u;
        for (uint32_t q = lane; q < npairs; q += 32) {
          const unsigned long long v = b0 + head + 2u * q;
          d2[q] = make_ulonglong2(v, v + 1);
        }
        if (((1024u - head) & 1u) && lane == 0) dst[1023] = b0 + 1023u;
      } else {
        for (uint32_t q = lane; q < 1024u; q += 32)
          if (o + q < cap) dst[q] = b0 + q;
      }
      o += 1024u;
      continue;
    }
    const uint32_t pc = __popc(mk);
    const uint32_t incl = warp_incl_scan_x(pc, lane);
    const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (tot == 0) continue;
    uint32_t j = incl - pc;
    const uint32_t u0 = w * wspan + 32u * i;
    while (mk) {
      const uint32_t b = __ffs(mk) - 1;
      mk &= mk - 1;
      sbuf[j++] = (uint16_t)(u0 + b);
    }
    __syncwarp();
    for (uint32_t q = lane; q < tot; q += 32)
      if (o + q < cap) pos[o + q] = (uint64_t)(pos_base + (int64_t)sbuf[q]);
    __syncwarp();
    o += tot;
  }
}

__global__ void __launch_bounds__(kExpandWarps * 32, 2) stage_expand_kernel(const uint8_t* stage,
                                                                        const unsigned long long* stage_used,
                                                                        uint64_t cap16, const uint16_t* wc,
                                                                        const uint64_t* tile_offsets, uint64_t* pos,
                                                                        uint64_t cap, unsigned long long* work) {
  extern __shared__ __align__(16) uint8_t xsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* cbuf = xsm + warp * kWarpSmem;                                    // the chunk
  uint64_t* rout = reinterpret_cast<uint64_t*>(cbuf + kChunkBytes);           // [kMaxRecs] output offsets
  uint32_t* rpre = reinterpret_cast<uint32_t*>(rout + kMaxRecs);              // [kMaxRecs + 1] list-element prefix
  uint16_t* roff = reinterpret_cast<uint16_t*>(rpre + kMaxRecs + 1);          // [kMaxRecs] record offsets (units)
  uint16_t* sbuf = roff + kMaxRecs;                                           // [1024] bitmap expansion
  const unsigned long long used = *stage_used < cap16 ? *stage_used : cap16;
  const uint64_t nchunks = (used + kStageChunk - 1) / kStageChunk;
  // chunks are fetched from a counter, not split statically: dispatch order keeps the set
  // of output regions being written at any time narrow (pool chunks are allocated in
  // tile order), which the HBM write path rewards (tools/wprobe.py: 7.4-7.6 TB/s for
  // counter-dispatched 32 KiB regions vs 6.2-6.3 for any static split; dense report
  // 1.78 -> 1.65 ms).  Splitting a chunk's records over several warps was slower.
  while (true) {
    unsigned long long ch = 0;
    if (lane == 0) ch = atomicAdd(work, 1ull);
    ch = __shfl_sync(0xFFFFFFFFu, ch, 0);
    if (ch >= nchunks) break;
    const uint64_t base16 = ch * kStageChunk;
    const uint32_t len16 = (uint32_t)(cap16 - base16 < kStageChunk ? cap16 - base16 : kStageChunk);
    const uint4* src = reinterpret_cast<const uint4*>(stage + base16 * 16u);
    uint4* dst = reinterpret_cast<uint4*>(cbuf);
#pragma unroll 8
    for (uint32_t i = lane; i < len16; i += 32) dst[i] = src[i];
    __syncwarp();
    uint32_t nrec = 0;
    if (lane == 0) {  // walk the chain of records up to the terminator (or the chunk's end)
      uint32_t o = 0;
      while (o < len16) {
        const uint32_t hw = reinterpret_cast<const uint32_t*>(cbuf + o * 16u)[3];
        const uint32_t c = hw & 0xFFFFu;
        if (c == 0) break;
        roff[nrec++] = (uint16_t)o;
        o += 1u + rec_data_bytes(c, rec_wspan(hw), is_list_record(hw)) / 16u;
      }
    }
    nrec = __shfl_sync(0xFFFFFFFFu, nrec, 0);
    __syncwarp();
    // output offset of each record: lane l takes records l, l + 32, ..., four at a time so
    // that four independent pairs of global loads are in flight
    for (uint32_t r0 = lane; r0 < nrec; r0 += 128) {
      uint4 v[4];
      uint64_t off[4];
      uint32_t wv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t r = r0 + 32u * u;
        if (r < nrec) {
          const uint4 h = *reinterpret_cast<const uint4*>(cbuf + roff[r] * 16u);
          wv[u] = (h.w >> 16) & 0xFFu;
          rpre[r] = is_list_record(h.w) ? (h.w & 0xFFFFu) : 0u;
          v[u] = reinterpret_cast<const uint4*>(wc)[h.z];
          off[u] = tile_offsets[h.z];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t r = r0 + 32u * u;
        if (r >= nrec) break;
        const uint32_t cw[8] = {v[u].x & 0xFFFFu, v[u].x >> 16, v[u].y & 0xFFFFu, v[u].y >> 16,
                                v[u].z & 0xFFFFu, v[u].z >> 16, v[u].w & 0xFFFFu, v[u].w >> 16};
        uint64_t pre = 0;
#pragma unroll
        for (uint32_t q = 0; q < 8; ++q)
          if (q < wv[u]) pre += cw[q];
        rout[r] = off[u] + pre;
      }
    }
    __syncwarp();
    // u16-list records, flattened: element e of the chunk's concatenated lists goes to
    // lane e mod 32, so a warp store covers 32 consecutive elements (1-3 records of a
    // sparse chunk) instead of one record's few positions
    uint32_t carry = 0;
    for (uint32_t b = 0; b < nrec; b += 32) {  // exclusive prefix of the list lengths
      const uint32_t v = b + lane < nrec ? rpre[b + lane] : 0u;
      const uint32_t incl = warp_incl_scan_x(v, lane);
      if (b + lane < nrec) rpre[b + lane] = carry + incl - v;
      carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
    if (lane == 0) rpre[nrec] = carry;
    __syncwarp();
    {
      uint32_t r = 0, r_beg = 0, r_end = nrec ? rpre[1] : 0u;
      bool fresh = true;
      uint64_t out0 = 0;
      int64_t base = 0;
      const uint16_t* L = nullptr;
      for (uint32_t e = lane; e < carry; e += 32) {
        while (e >= r_end) {  // lanes only move forward through the records
          ++r;
          r_end = rpre[r + 1];
          fresh = true;
        }
        if (fresh) {
          const uint8_t* rec = cbuf + roff[r] * 16u;
          const uint2 hb = *reinterpret_cast<const uint2*>(rec);
          base = (int64_t)(((uint64_t)hb.y << 32) | hb.x);
          L = reinterpret_cast<const uint16_t*>(rec + kRecHeader);
          out0 = rout[r];
          r_beg = rpre[r];
          fresh = false;
        }
        const uint32_t i = e - r_beg;
        if (out0 + i < cap) pos[out0 + i] = (uint64_t)(base + (int64_t)L[i]);
      }
    }
    for (uint32_t r = 0; r < nrec; ++r) {  // bitmap records (no list elements)
      const uint64_t out = rout[r];
      if (rpre[r + 1] == rpre[r] && out < cap) write_bitmap(cbuf + roff[r] * 16u, out, pos, cap, sbuf, lane);
    }
    __syncwarp();  // cbuf / rout are reused for the next chunk
  }
}

}  // namespace

cudaError_t launch_stage_expand(const uint8_t* stage, const unsigned long long* stage_used, uint64_t stage_cap16,
                                const uint16_t* wc, const uint64_t* tile_offsets, uint64_t* pos, uint64_t cap,
                                unsigned long long* work, int num_sms, cudaStream_t st) {
  if (stage_cap16 == 0) return cudaSuccess;
  const size_t smem = (size_t)kExpandWarps * kWarpSmem;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  static bool attr[64] = {};  // per device context; benign race: idempotent
  if (!attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(stage_expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[dev] = true;
  }
  const uint64_t max_chunks = (stage_cap16 + kStageChunk - 1) / kStageChunk;
  const uint64_t want = (max_chunks + kExpandWarps - 1) / kExpandWarps;
  const uint64_t lim = (uint64_t)num_sms * 2;  // 2 CTAs of 8 warps per SM (shared memory)
  const int grid = (int)(want < lim ? want : lim);
  stage_expand_kernel<<<grid, kExpandWarps * 32, smem, st>>>(stage, stage_used, stage_cap16, wc, tile_offsets, pos,
                                                             cap, work);
  return cudaGetLastError();
}

}  // namespace smgpu
