// scan.cu -- exclusive prefix over per-tile match counts (reporting, A8).
#include <cub/device/device_scan.cuh>

#include "launch.h"

namespace smgpu {

cudaError_t exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, void* temp, size_t* temp_bytes,
                               cudaStream_t st) {
  return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, in, out, static_cast<int>(count), st);
}

}  // namespace smgpu
