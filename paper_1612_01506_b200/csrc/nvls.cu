// nvls.cu -- NEXT-4: the all-reduce of per-rank pattern counts through NVLink SHARP
// (NVLS): each rank adds its local counts to an NVLink multicast address with one
// multimem.red per pattern; the switch applies the add to every rank's bound copy, so
// after all ranks' launches every copy holds the global sums -- no NCCL call.
// Kept out of the search kernel: inline-asm multimem there is a convergent operation
// that forced reconvergence barriers into the hot loop.
#include "device_util.cuh"
#include "launch.h"

namespace smgpu {
namespace {
__global__ void nvls_add_kernel(const uint64_t* __restrict__ local, uint64_t* mc, uint64_t P) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < P; i += (uint64_t)gridDim.x * blockDim.x)
    if (local[i]) multimem_red_add_u64(mc + i, (unsigned long long)local[i]);
}
}  // namespace

cudaError_t launch_nvls_add(const uint64_t* local, uint64_t* mc, uint64_t P, cudaStream_t st) {
  if (P == 0) return cudaSuccess;
  const uint64_t want = (P + 255) / 256;
  const int grid = (int)(want < 1024 ? want : 1024);
  nvls_add_kernel<<<grid, 256, 0, st>>>(local, mc, P);
  return cudaGetLastError();
}
}  // namespace smgpu
