// search_filter.cu -- instantiations of the FILTER strategy (see search_impl.cuh).
#include "search_dispatch.cuh"

namespace smgpu {
cudaError_t launch_search_filter(const HostLaunch& L, cudaStream_t st) { return launch_strategy<kFilter>(L, st); }
}  // namespace smgpu
