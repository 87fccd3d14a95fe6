// search.cuh -- kernel-side description of one search launch.
#pragma once
#include <cstdint>

namespace smgpu {

constexpr int kConsumerWarps = 8;                        // warps comparing text
constexpr int kThreads = (kConsumerWarps + 1) * 32;      // + 1 TMA producer warp
constexpr int kChunk = 16;                               // alignments per lane-chunk
constexpr int kLanesPerTilePass = kConsumerWarps * 32;   // lanes sharing a tile
constexpr int kMaxStages = 8;
constexpr int kMaxCPL = 8;                               // chunks per lane per tile (tile <= 32 KiB)
constexpr int kGroup = 8;                                // FILTER: chunk-rows per queue fill
constexpr int kQueueLen = 32 * kGroup;                   // FILTER: queue entries per warp
constexpr uint32_t kLaneVerifyMaxM = 34;                 // FILTER: per-lane verification up to this m
// shared-memory layout: [full/empty mbarriers][warp totals [2][W]][queue chunk ids u16 [W][kQueueLen]][table][ring]
constexpr uint32_t kWarpTotOff = 2 * kMaxStages * 8;
constexpr uint32_t kQueueOff = kWarpTotOff + 2 * kConsumerWarps * 4;
constexpr uint32_t kTblOff = kQueueOff + kConsumerWarps * kQueueLen * 2;

enum Strategy : int { kFilter = 1, kBlock = 2 };
enum Epilogue : int { kEpiCount = 0, kEpiTileCount = 1, kEpiWrite = 2 };

// Everything about a launch except the pattern table.  All byte offsets are
// relative to `base` = align_down(t, 16); the text occupies offsets
// [delta, delta + n).  Alignment offset x <-> 0-based position x - delta.
struct SearchArgs {
  const uint8_t* base;
  uint64_t delta;         // t - base (0..15)
  uint64_t n;             // text length
  uint64_t A;             // number of alignments, n - m + 1  (n >= m)
  uint64_t k_begin;       // first tile index (tile k covers [kT, kT+T) in its space)
  uint64_t ntiles;        // tiles k_begin .. k_begin + ntiles - 1
  uint64_t edge_lo;       // tiles ti < edge_lo start before the first alignment
  uint64_t edge_hi;       // tiles ti >= edge_hi end after the last alignment
  uint32_t m;
  uint32_t r;             // peeling factor (block strategy), 1 <= r <= m
  uint32_t a1;            // pattern offset of pi(1)       (filter strategy)
  uint32_t bc1;           // p[pi(1)] * 0x01010101          (filter strategy)
  uint32_t s2;            // pre + off(pi(2)) - a1: buffer offset of pi(2)'s byte for u = 0 (filter)
  uint32_t bc2;           // p[pi(2)] * 0x01010101          (filter strategy, m >= 2)
  uint32_t tile;          // T, multiple of 16 * kLanesPerTilePass
  uint32_t pre;           // buffer bytes before the tile (multiple of 16)
  uint32_t stage_len;     // bytes a stage holds = T + pre + post (multiple of 16)
  uint32_t stage_stride;  // smem stride between stages (multiple of 128)
  uint32_t stages;        // ring depth
  uint32_t ring_off;      // smem byte offset of stage 0
  uint64_t* count_out;    // kEpiCount: device u64 (accumulated with atomics; zeroed by host)
  uint64_t* tile_counts;  // kEpiTileCount: u64[ntiles] (zeroed by host); kEpiWrite: unused
  const uint64_t* tile_offsets;  // kEpiWrite: exclusive prefix, ntiles + 1 entries
  uint64_t* pos;          // kEpiWrite: output positions
  uint64_t cap;           // kEpiWrite: capacity of pos
};

// Pattern in comparison order: e[k] = off(pi(k)) | p[pi(k)] << 16.
template <int MAXM>
struct PatternTable {
  uint32_t e[MAXM];
};

}  // namespace smgpu
