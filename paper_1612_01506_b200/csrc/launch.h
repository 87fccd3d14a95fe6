// launch.h -- internal host-side entry points of the kernels (not part of the ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "search.cuh"

namespace smgpu {

cudaError_t launch_hist(const uint8_t* t, uint64_t n, uint64_t* d_hist, int num_sms, cudaStream_t st);

// table: m entries e[k] = off(pi(k)) | p[pi(k)] << 16
cudaError_t launch_search(const SearchArgs& a, const uint32_t* table, int strategy, int epilogue, int cpl,
                          int grid, size_t smem_bytes, cudaStream_t stream);

cudaError_t exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, void* temp, size_t* temp_bytes,
                               cudaStream_t st);

}  // namespace smgpu
