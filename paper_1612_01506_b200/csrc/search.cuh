// search.cuh -- kernel-side description of one search launch (a batch of
// patterns over one device text; each pattern is a full pass over the text).
#pragma once
#include <cstdint>

namespace smgpu {

constexpr int kConsumerWarps = 8;                        // warps comparing text
constexpr int kThreads = (kConsumerWarps + 1) * 32;      // + 1 TMA producer warp
constexpr int kLanesPerTilePass = kConsumerWarps * 32;   // lanes sharing a tile
constexpr int kMaxStages = 8;
constexpr int kGroup = 8;                                // FILTER: chunk-rows per queue fill
constexpr int kQueueLen = 32 * kGroup;                   // FILTER: queue entries per warp
constexpr uint32_t kLaneVerifyMaxM = 34;                 // FILTER: per-lane verification up to this m
constexpr int kMaxBatch = 64;                            // patterns per launch
constexpr int kListCap = 512;                            // reporting (overflow pass): buffered positions per warp and tile
constexpr int kTableSmall = 256;                         // pattern-table capacities (u32 entries)
constexpr int kTableMid = 2048;                          // (the launch cost grows with the parameter block:
                                                         //  ~10 us at 8 KiB, ~27 us at 32 KiB on B200)
constexpr int kTableLarge = 6400;                        // with 64 descriptors: fills the 32 KiB parameter space
constexpr int kBatchTableWords = kTableLarge;            // batching: table entries per launch

// shared-memory layout: [full/empty mbarriers][warp totals [2][W]][queue chunk ids u16 [W][kQueueLen]]
//                       [dispatched item per stage u32][PACKED code buffers][ring]   (the pattern tables stay in the kernel parameters)
constexpr uint32_t kWarpTotOff = 2 * kMaxStages * 8;
constexpr uint32_t kQueueOff = kWarpTotOff + 2 * kConsumerWarps * 4;
// [kMaxStages] uint4 dispatched items {w, pattern k, tile ti, edge}: the producer maps w once
// per item, the 8 consumer warps read the result with one LDS.128
constexpr uint32_t kTixOff = kQueueOff + kConsumerWarps * kQueueLen * 2;
static_assert(kTixOff % 16 == 0, "tix slots are read as uint4");
constexpr uint32_t kTblOff = kTixOff + kMaxStages * 16;                     // end of the fixed region
constexpr uint32_t kNoItem = 0xFFFFFFFFu;  // dispatched-item sentinel: the producer is done

// kPackedB: b-bit codes; kPair: FILTER whose chunk test covers pi(1) and pi(2) together
// kPackedBPre: PACKED reading a code array packed once per call (pack_text_kernel) instead
// of packing every tile (NEXT-3: the per-symbol codes memoised at text scope)
enum Strategy : int { kFilter = 1, kBlock = 2, kPacked1 = 3, kPacked2 = 4, kPair = 5, kPacked1Pre = 6, kPacked2Pre = 7 };
__host__ __device__ constexpr bool is_packed(int s) { return s == kPacked1 || s == kPacked2 || s >= kPacked1Pre; }
__host__ __device__ constexpr bool is_prepacked(int s) { return s >= kPacked1Pre; }
__host__ __device__ constexpr int code_bits(int s) { return (s == kPacked2 || s == kPacked2Pre) ? 2 : 1; }
// kEpiCount: per-pattern counts.  kEpiStage: reporting pass 1 -- per-(pattern, tile) counts
// plus the tile's matches staged compactly in global memory (per-warp u16 offset lists
// or bitmaps), expanded into positions by stage_expand_kernel after the scan: the
// text is read once.  kEpiWrite: reporting fallback for the tiles whose staging did
// not fit the pool (overflow queue): recompute from the text, write positions.
// kEpiCountMc: kEpiCount + the NEXT-4 last-CTA epilogue (multimem.red of the launch's
// counts to an NVLink multicast address, LaunchArgs::mc_base) -- a separate instantiation.
enum Epilogue : int { kEpiCount = 0, kEpiStage = 1, kEpiWrite = 2, kEpiCountMc = 3 };
__host__ __device__ constexpr bool is_count_epi(int e) { return e == kEpiCount || e == kEpiCountMc; }

// Staged reporting (kEpiStage): every compare warp with matches in a work item writes
// one self-describing record into its own chunk of the staging pool (kStageChunk
// 16-B units per chunk, grabbed with one global atomic; records packed back to back,
// a zero header terminates a chunk's records):
//   header (16 B): i64 pos_base (0-based position of tile-relative alignment u = 0,
//                  shard offset included), u32 item, u16 cnt, u8 warp, then bits 24-25
//                  log2(CPL) and bit 31 = bitmap record;
//   data: a list record (cnt <= list_max and 2 cnt < wspan / 8, wspan = 512 CPL
//         alignments per warp) holds the ascending u16 list of the tile-relative
//         alignments u (padded to 16 B); a bitmap record the warp's bitmap, wspan / 16
//         u16 words, bit b of word i <-> u = warp wspan + 16 i + b.
// and posts cnt into wc[item][warp] (u16 x 8 per item, zero-initialised): the scan of
// the per-item sums gives each item's output offset, wc its warps' order inside it.
constexpr uint32_t kRecHeader = 16;
constexpr uint32_t kStageChunk = 512;   // 16-B units (8 KiB) >= largest record (528 B) + terminator
constexpr uint32_t kRecBitmap = 1u << 31;  // header word 3: bitmap record
__host__ __device__ inline bool rec_is_list(uint32_t cnt, uint32_t wspan, uint32_t list_max) {
  return cnt <= list_max && 2u * cnt < wspan / 8u;
}
__host__ __device__ inline uint32_t rec_data_bytes(uint32_t cnt, uint32_t wspan, bool list) {
  if (cnt == 0) return 0;
  return list ? ((2u * cnt + 15u) & ~15u) : wspan / 8u;
}

// One pattern of a launch.  Byte offsets are relative to `base` = align_down(t, 16);
// the text occupies offsets [delta, delta + n); alignment offset x <-> position x - delta.
// Tile k covers tile-relative positions u in [kT, kT+T): FILTER u indexes the
// pi(1)-bytes (alignment x = kT + u - a1), BLOCK the alignments (x = kT + u).
struct PatDesc {
  uint64_t A;          // alignments counted (n - m + 1, or fewer when limited)
  uint64_t k_begin;    // first tile index
  uint64_t ntiles;     // tiles k_begin .. k_begin + ntiles - 1
  uint64_t work_end;   // this pattern's work items are [work_end - ntiles, work_end)
  uint64_t edge_lo;    // tiles ti < edge_lo start before the first alignment
  uint64_t edge_hi;    // tiles ti >= edge_hi end after the last alignment
  uint64_t* count_out; // kEpiCount / kEpiStage: device u64 (accumulated with atomics; zeroed by host)
  uint64_t item_base;  // reporting: index of this pattern's first tile in wc / tile_offsets
  uint32_t m;
  uint32_t r;          // peeling factor (BLOCK), 1 <= r <= m
  uint32_t a1;         // pattern offset of pi(1) (FILTER)
  uint32_t bc1;        // p[pi(1)] * 0x01010101 (FILTER)
  uint32_t s2;         // pre + off(pi(2)) - a1: buffer offset of pi(2)'s byte for u = 0 (FILTER, m >= 2)
  uint32_t bc2;        // p[pi(2)] * 0x01010101 (FILTER, m >= 2)
  uint32_t pre;        // buffer bytes before the tile (multiple of 16)
  uint32_t stage_len;  // bytes the tile's buffer holds = T + pre + post (multiple of 16)
  uint32_t tbl;        // index of this pattern's first entry in LaunchParams::e
  uint32_t flags;       // bit 0: tiles visited in descending order (alternating passes share the L2-resident
                       // seam); bits 8..15 (PACKED): r1 = the first r1 peeled steps read only the register
                       // window (the host moves them to the front of the peeled steps, which all run)
};

struct LaunchArgs {
  const uint8_t* base;
  uint64_t delta;
  uint64_t n;
  uint64_t total_work;       // sum of ntiles over the batch
  uint32_t tile;             // T, multiple of 16 * kLanesPerTilePass
  uint32_t stage_stride;     // smem stride between stages (multiple of 128)
  uint32_t stages;           // ring depth
  uint32_t ring_off;         // smem byte offset of stage 0
  uint32_t npat;             // patterns in the batch
  uint32_t tbl_words;        // table entries
  uint32_t code_shift;       // PACKED: code(x) = (x >> code_shift) & (2^b - 1), injective on the text's symbols
  uint32_t l2_policy;        // TMA loads: 0 evict_first, 1 evict_normal, 2 evict_last (performance only)
  uint32_t wait_ns;          // consumers' full-stage wait: suspend-time hint (0 = spin)
  uint32_t pack_off;         // PACKED: smem byte offset of the double-buffered code array
  uint32_t pack_bytes;       // PACKED: bytes of one code buffer
  const uint8_t* codes;      // kPackedBPre: the code array of the text (base-relative alignment x <-> code bits
                             // [b x, b x + b) of the array), 16-B aligned, zero past the text
  uint32_t list_off;         // reporting: smem byte offset of the per-warp position lists [W][kListCap] u16
  uint16_t* wc;              // kEpiStage: per item u16[kConsumerWarps] match counts (zeroed by host)
  uint8_t* stage;            // kEpiStage: staging pool (records)
  unsigned long long* stage_used;  // kEpiStage: pool chunk bump pointer (16-B units, zeroed by host)
  uint64_t stage_cap16;      // kEpiStage: pool size in 16-B units
  uint32_t* ovf_bits;        // kEpiStage: per item, set once its first warp failed to stage (zeroed by host)
  uint32_t* ovf_items;       // kEpiStage / kEpiWrite: this launch's overflow queue (items)
  uint32_t* ovf_n;           // kEpiStage / kEpiWrite: its length (zeroed by host)
  const uint64_t* tile_offsets;  // kEpiWrite: exclusive prefix of the per-item counts (patterns in caller order)
  uint64_t* pos;             // kEpiWrite: output positions
  uint64_t cap;              // kEpiWrite: capacity of pos
  uint64_t pos_offset;       // kEpiStage / kEpiWrite: added to every position (a shard's first owned position)
  uint32_t list_max;         // kEpiStage: a warp with at most this many matches stages a list record, more a bitmap
  unsigned long long* ctr;   // instrumented build (SMGPU_COUNTERS) only: device u64[kCounters], else unused
  unsigned long long* work_ctr;  // count / stage: non-null = work items are dispatched from this zeroed
                                 // counter (the producer fetches, the consumers read the stage's item)
  const uint32_t* guard;     // device flag set by pack_text_kernel when a text byte lies outside the symbol
                             // set the code field was chosen for (a caller histogram that is not t's)
  uint32_t guard_mode;       // 0: always run; kGuardClear: run only if *guard == 0 (PACKED on a caller
                             // histogram); kGuardSet: run only if *guard != 0 (its byte-compare fallback)
  // NEXT-4 (kEpiCountMc): after every CTA's atomics, the last CTA to finish
  // (done_ctr, zeroed by the host) adds each pattern's count, read from count_out, to
  // mc_base + (count_out - local_base) with one multimem.red (NVLink multicast: the
  // switch adds it to every rank's copy).  mc_emulate: plain atomicAdd instead (tests on
  // a box without multicast: same protocol, unicast address).
  uint64_t* mc_base;
  const uint64_t* local_base;
  unsigned int* done_ctr;
  uint32_t mc_emulate;
};
constexpr uint32_t kGuardClear = 1, kGuardSet = 2;

// Compare-step counters of the instrumented build (libsmgpu_counters.so, NEXT-2):
enum Counter : int {
  kCtrWarpTiles = 0,     // (warp, work item) pairs processed
  kCtrBlocks = 1,        // BLOCK / PACKED: warp-blocks (512 CPL alignments) holding >= 1 valid alignment
  kCtrSteps = 2,         // BLOCK / PACKED: SIMDcompare steps (peeled + ordered loop) executed in those blocks
  kCtrChunks = 3,        // FILTER: 16-alignment chunks whose pi(1)-bytes were tested (phase A)
  kCtrQueued = 4,        // FILTER: chunks holding p[pi(1)] (queued for phase B)
  kCtrSurvivors = 5,     // FILTER: valid alignments matching pi(1) and pi(2) (entering verification)
  kCtrVerify = 6,        // FILTER: pattern positions compared while verifying survivors
  kCtrAlphaEff = 7,      // BLOCK / PACKED: alignments per warp-block (max)
  kCounters = 8
};

// Kernel parameters: everything per launch, no __constant__ state, so launches on
// different streams never race.  Table entry = off(pi(k)) | p[pi(k)] << 16
// (PACKED: the symbol's b-bit code instead of the byte).
template <int CAP>
struct LaunchParams {
  LaunchArgs a;
  PatDesc d[kMaxBatch];
  uint32_t e[CAP];
};
static_assert(sizeof(LaunchParams<kTableLarge>) <= 32764, "kernel parameter space is 32764 bytes on sm_100a");

}  // namespace smgpu
