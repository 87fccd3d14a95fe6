// scan.cu -- exclusive prefix over per-item match counts (reporting, A8): the output
// offset of every (pattern, tile) work item in the concatenated position array.
//
// Single pass, decoupled look-back: each CTA takes the next tile of kScanTile items
// (tile order = the order CTAs start, from a counter, so every predecessor is running
// or done), sums each item's u16 x 8 warp counts, scans the tile in shared memory,
// publishes its aggregate, then one warp walks back over the predecessors' published
// aggregates / inclusive prefixes 32 at a time until it meets an inclusive prefix.
// Status word per tile: bits 62-63 flag (0 not yet, 1 aggregate, 2 inclusive prefix),
// bits 0-61 the value (a count of positions: < 2^62).  Reads every item once (16 B),
// writes its u64 offset once.
#include "launch.h"

namespace smgpu {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanPer = 8;                                // items per thread
constexpr int kScanTile = kScanThreads * kScanPer;         // 2048 items per CTA
constexpr uint64_t kFlagA = 1ull << 62, kFlagP = 2ull << 62, kValMask = kFlagA - 1;
static_assert(kConsumerWarps == 8, "one uint4 of u16 warp counts per item");

__host__ __device__ constexpr uint32_t pad(uint32_t k) { return k + (k >> 5); }  // conflict-free transposition

__device__ __forceinline__ uint64_t ld_status(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__global__ void __launch_bounds__(kScanThreads) scan_wc_kernel(const uint4* __restrict__ wc, uint64_t* __restrict__ out,
                                                               uint64_t items, unsigned long long* status,
                                                               unsigned int* tile_ctr) {
  __shared__ uint32_t s_v[pad(kScanTile)];
  __shared__ uint64_t s_o[pad(kScanTile)];
  __shared__ uint64_t s_warp[kScanThreads / 32];
  __shared__ uint64_t s_prefix;
  __shared__ uint32_t s_tile;
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * (uint64_t)kScanTile;
  // coalesced loads: item base + i * 256 + t
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    const uint64_t idx = base + (uint64_t)i * kScanThreads + t;
    uint32_t v = 0;
    if (idx < items) {
      const uint4 w = wc[idx];
      v = (w.x & 0xFFFFu) + (w.x >> 16) + (w.y & 0xFFFFu) + (w.y >> 16) + (w.z & 0xFFFFu) + (w.z >> 16) +
          (w.w & 0xFFFFu) + (w.w >> 16);
    }
    s_v[pad(i * kScanThreads + t)] = v;
  }
  __syncthreads();
  // thread t owns items t * kScanPer .. + kScanPer - 1 of the tile
  uint32_t mine[kScanPer];
  uint64_t sum = 0;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    mine[j] = s_v[pad(t * kScanPer + j)];
    sum += mine[j];
  }
  // block exclusive scan of the per-thread sums
  uint64_t incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if ((int)lane >= d) incl += u;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint64_t wpre = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    const uint64_t x = s_warp[w];
    if (w < (int)warp) wpre += x;
    agg += x;
  }
  const uint64_t texcl = wpre + incl - sum;  // exclusive prefix of thread t inside the tile
  // look-back: the tile's exclusive prefix over all earlier tiles
  if (warp == 0) {
    uint64_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(status) = kFlagP | agg;
    } else {
      if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(status + tile) = kFlagA | agg;
      int64_t j = (int64_t)tile - 1;  // predecessor read by lane 0 (lane l reads j - l)
      while (true) {
        const int64_t q = j - (int64_t)lane;
        uint64_t st = q >= 0 ? ld_status(status + q) : kFlagP;  // before tile 0: an empty inclusive prefix
        const uint32_t pmask = __ballot_sync(0xFFFFFFFFu, (st >> 62) == 2u);
        const uint32_t span = pmask ? (pmask & (0u - pmask)) * 2u - 1u : 0xFFFFFFFFu;  // lanes up to the first P
        if (__any_sync(0xFFFFFFFFu, ((span >> lane) & 1u) && (st >> 62) == 0u)) continue;  // not all published
        uint64_t v = ((span >> lane) & 1u) ? (st & kValMask) : 0;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
        prefix += v;
        if (pmask) break;
        j -= 32;
      }
      if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(status + tile) = kFlagP | (prefix + agg);
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  uint64_t run = s_prefix + texcl;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    s_o[pad(t * kScanPer + j)] = run;
    run += mine[j];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    const uint64_t idx = base + (uint64_t)i * kScanThreads + t;
    if (idx < items) out[idx] = s_o[pad(i * kScanThreads + t)];
  }
}

}  // namespace

cudaError_t exclusive_scan_wc(const uint16_t* wc, uint64_t* out, uint64_t items, void* temp, size_t* temp_bytes,
                              cudaStream_t st) {
  const uint64_t tiles = (items + kScanTile - 1) / kScanTile;
  const size_t need = (size_t)(tiles * 8 + 16);
  if (!temp) {
    *temp_bytes = need;
    return cudaSuccess;
  }
  if (items == 0) return cudaSuccess;
  if (*temp_bytes < need || tiles >= (1ull << 31)) return cudaErrorInvalidValue;
  unsigned long long* status = static_cast<unsigned long long*>(temp);
  unsigned int* ctr = reinterpret_cast<unsigned int*>(status + tiles);
  cudaError_t e = cudaMemsetAsync(temp, 0, need, st);
  if (e != cudaSuccess) return e;
  scan_wc_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(reinterpret_cast<const uint4*>(wc), out, items, status,
                                                           ctr);
  return cudaGetLastError();
}

}  // namespace smgpu
