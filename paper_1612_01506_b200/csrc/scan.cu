// scan.cu -- exclusive prefix over per-item match counts (reporting, A8).
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "launch.h"

namespace smgpu {
namespace {
// an item's match count = the sum of its compare warps' counts (u16 x 8 = one uint4)
struct SumWarpCounts {
  __host__ __device__ __forceinline__ uint64_t operator()(const uint4& v) const {
    return (uint64_t)(v.x & 0xFFFFu) + (v.x >> 16) + (v.y & 0xFFFFu) + (v.y >> 16) + (v.z & 0xFFFFu) +
           (v.z >> 16) + (v.w & 0xFFFFu) + (v.w >> 16);
  }
};
static_assert(kConsumerWarps == 8, "one uint4 of u16 warp counts per item");
}  // namespace

cudaError_t exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, void* temp, size_t* temp_bytes,
                               cudaStream_t st) {
  return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, in, out, static_cast<int>(count), st);
}

cudaError_t exclusive_scan_wc(const uint16_t* wc, uint64_t* out, uint64_t items, void* temp, size_t* temp_bytes,
                              cudaStream_t st) {
  cub::TransformInputIterator<uint64_t, SumWarpCounts, const uint4*> it(reinterpret_cast<const uint4*>(wc),
                                                                        SumWarpCounts());
  return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, it, out, static_cast<int>(items), st);
}

}  // namespace smgpu
