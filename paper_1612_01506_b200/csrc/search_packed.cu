// search_packed.cu -- instantiations of the PACKED strategy (b-bit codes, see search_impl.cuh).
#include "search_dispatch.cuh"

namespace smgpu {
cudaError_t launch_search_packed(const HostLaunch& L, cudaStream_t st) {
  if (L.strategy == kPacked2) return launch_strategy<kPacked2>(L, st);
  return launch_strategy<kPacked1>(L, st);
}
}  // namespace smgpu
