// search_kernel.cu -- strategy dispatch (kernels live in search_impl.cuh).
#include "launch.h"

namespace smgpu {

cudaError_t launch_search_filter(const SearchArgs& a, const uint32_t* table, int epilogue, int cpl, int grid,
                                 size_t smem_bytes, cudaStream_t stream);
cudaError_t launch_search_block(const SearchArgs& a, const uint32_t* table, int epilogue, int cpl, int grid,
                                size_t smem_bytes, cudaStream_t stream);

cudaError_t launch_search(const SearchArgs& a, const uint32_t* table, int strategy, int epilogue, int cpl,
                          int grid, size_t smem_bytes, cudaStream_t stream) {
  if (strategy == kFilter) return launch_search_filter(a, table, epilogue, cpl, grid, smem_bytes, stream);
  return launch_search_block(a, table, epilogue, cpl, grid, smem_bytes, stream);
}

}  // namespace smgpu
