// launch.h -- internal host-side entry points of the kernels (not part of the ABI).
#pragma once
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "search.cuh"

namespace smgpu {

// A planned search launch: one strategy, one epilogue, a batch of <= kMaxBatch
// patterns whose pattern tables total <= kTableLarge entries.
struct HostLaunch {
  LaunchArgs a;
  std::vector<PatDesc> d;
  std::vector<uint32_t> e;
  int strategy = kFilter;
  int epilogue = kEpiCount;
  int cpl = 8;
  int grid = 1;
  size_t smem = 0;
};

cudaError_t launch_hist(const uint8_t* t, uint64_t n, uint64_t* d_hist, int num_sms, cudaStream_t st);

cudaError_t launch_search(const HostLaunch& L, cudaStream_t stream);

// Reporting: expand the staged records of the pool (chunks [0, min(*stage_used,
// stage_cap16)) into positions pos[tile_offsets[item] + warps before + j] (< cap),
// see search.cuh.
cudaError_t launch_stage_expand(const uint8_t* stage, const unsigned long long* stage_used, uint64_t stage_cap16,
                                const uint16_t* wc, const uint64_t* tile_offsets, uint64_t* pos, uint64_t cap,
                                unsigned long long* work /* zeroed chunk counter */, int num_sms, cudaStream_t st);

// NEXT-3: the text's b-bit code array (code(x) = (x >> shift) & (2^b - 1)), base-relative
// alignment x <-> bits [b x, b x + b); code_bytes (multiple of 16) of it, zero past the text.
// bad != nullptr: also sets *bad (device u32, zeroed by the caller) if some text byte is
// not one of the four bytes of syms (the symbols the code field was chosen for).
cudaError_t launch_pack_text(const uint8_t* base, uint64_t delta, uint64_t n, uint32_t shift, int b, uint8_t* codes,
                             uint64_t code_bytes, uint32_t syms, uint32_t* bad, int num_sms, cudaStream_t st);

// exclusive prefix over items of the sum of wc[item][0..8) (u16 warp counts); temp == nullptr:
// *temp_bytes = the scratch it needs (single-pass decoupled look-back, scan.cu; 2 launches:
// a memset of the tile status words and the scan)
cudaError_t exclusive_scan_wc(const uint16_t* wc, uint64_t* out, uint64_t items, void* temp, size_t* temp_bytes,
                              cudaStream_t st);


}  // namespace smgpu
