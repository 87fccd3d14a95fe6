// search_block.cu -- instantiations of the BLOCK strategy (Alg. 4, see search_impl.cuh).
#include "search_dispatch.cuh"

namespace smgpu {
cudaError_t launch_search_block(const SearchArgs& a, const uint32_t* table, int epilogue, int cpl, int grid,
                                size_t smem_bytes, cudaStream_t stream) {
  return launch_strategy<kBlock>(a, table, epilogue, cpl, grid, smem_bytes, stream);
}
}  // namespace smgpu
