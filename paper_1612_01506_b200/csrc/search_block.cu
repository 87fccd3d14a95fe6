// search_block.cu -- instantiations of the BLOCK strategy (Alg. 4, see search_impl.cuh).
#include "search_dispatch.cuh"

namespace smgpu {
cudaError_t launch_search_block(const HostLaunch& L, cudaStream_t st) { return launch_strategy<kBlock>(L, st); }
}  // namespace smgpu
