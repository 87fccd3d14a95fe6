// search_filter.cu -- instantiations of the FILTER strategy (see search_impl.cuh).
#include "search_dispatch.cuh"

namespace smgpu {
cudaError_t launch_search_filter(const SearchArgs& a, const uint32_t* table, int epilogue, int cpl, int grid,
                                 size_t smem_bytes, cudaStream_t stream) {
  return launch_strategy<kFilter>(a, table, epilogue, cpl, grid, smem_bytes, stream);
}
}  // namespace smgpu
