// search_pair.cu -- instantiations of the PAIR strategy (see search_impl.cuh).
#include "search_dispatch.cuh"

namespace smgpu {
cudaError_t launch_search_pair(const HostLaunch& L, cudaStream_t st) { return launch_strategy<kPair>(L, st); }
}  // namespace smgpu
