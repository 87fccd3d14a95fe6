// search_kernel.cu -- strategy dispatch (kernels live in search_impl.cuh).
#include "launch.h"

namespace smgpu {

cudaError_t launch_search_filter(const HostLaunch& L, cudaStream_t st);
cudaError_t launch_search_block(const HostLaunch& L, cudaStream_t st);
cudaError_t launch_search_packed(const HostLaunch& L, cudaStream_t st);
cudaError_t launch_search_pair(const HostLaunch& L, cudaStream_t st);
cudaError_t launch_search_packed_pre(const HostLaunch& L, cudaStream_t st);

cudaError_t launch_search(const HostLaunch& L, cudaStream_t st) {
  if (L.strategy == kFilter) return launch_search_filter(L, st);
  if (L.strategy == kBlock) return launch_search_block(L, st);
  if (L.strategy == kPair) return launch_search_pair(L, st);
  if (is_prepacked(L.strategy)) return launch_search_packed_pre(L, st);
  return launch_search_packed(L, st);
}

}  // namespace smgpu
