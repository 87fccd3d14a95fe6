// hist_kernel.cu -- A1: device byte histogram of the text, hist[c] = #{x : t[x] = c}.
// The paper takes symbol frequencies "from some relevant corpus"
// and orders comparisons by "their probabilities in the text"; the
// north star reads this as the histogram of t itself (reading R10).
//
// Persistent grid; 16-B streaming loads (ld.global.cs), 4 in flight per
// thread; per-warp privatised u32 bins in shared memory (one ATOMS.POPC.INC per byte: lanes
// incrementing the same bin are combined by the hardware); one u64 atomic per (block, bin).
// Bound: shared-memory atomic throughput, not HBM -- random bytes spread a warp's 32
// increments over random banks (~3.5-way conflicts): 2.6 TB/s on uniform bytes, 5.3 TB/s on
// skewed or periodic text (tools/hist_probe.py: bin replicas per lane group and 4 or 16
// warps per block were slower).  Once per text, amortised over every pattern pass.
#include "device_util.cuh"
#include "launch.h"

namespace smgpu {

constexpr int kHistWarps = 8;

__global__ void __launch_bounds__(kHistWarps * 32) hist_kernel(const uint8_t* __restrict__ t, uint64_t n,
                                                              unsigned long long* __restrict__ hist) {
  __shared__ uint32_t sh[kHistWarps][256];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kHistWarps * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  uint32_t* h = sh[warp];

  const uintptr_t ta = reinterpret_cast<uintptr_t>(t);
  const uint64_t head = ((16 - (ta & 15)) & 15) < n ? ((16 - (ta & 15)) & 15) : n;  // bytes before 16-B alignment
  const uint64_t nvec = (n - head) / 16;
  const uint4* v = reinterpret_cast<const uint4*>(t + head);

  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  SMGPU_DCHECK(head <= n && head + nvec * 16 <= n);
  // 4 loads in flight per thread per iteration (2: -7 to -10 %, tools/hist_probe.py; the
  // L2::cache_hint evict-first form of the search kernel's loads: -10 % here)
  for (; i + 3 * stride < nvec; i += 4 * stride) {
    uint4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = __ldcs(v + i + u * stride);  // ld.global.cs (evict-first)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t w[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        atomicAdd(&h[w[k] & 0xFF], 1u);
        atomicAdd(&h[(w[k] >> 8) & 0xFF], 1u);
        atomicAdd(&h[(w[k] >> 16) & 0xFF], 1u);
        atomicAdd(&h[w[k] >> 24], 1u);
      }
    }
  }
  for (; i < nvec; i += stride) {
    const uint4 a = __ldcs(v + i);
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      atomicAdd(&h[w[k] & 0xFF], 1u);
      atomicAdd(&h[(w[k] >> 8) & 0xFF], 1u);
      atomicAdd(&h[(w[k] >> 16) & 0xFF], 1u);
      atomicAdd(&h[w[k] >> 24], 1u);
    }
  }
  // ragged head / tail bytes (< 16 each), block 0 only
  if (blockIdx.x == 0) {
    const uint64_t tail0 = head + nvec * 16;
    for (uint64_t x = threadIdx.x; x < head; x += blockDim.x) atomicAdd(&h[ldg_u8_nc(t + x)], 1u);
    for (uint64_t x = tail0 + threadIdx.x; x < n; x += blockDim.x) atomicAdd(&h[ldg_u8_nc(t + x)], 1u);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 256; c += blockDim.x) {
    uint64_t s = 0;
#pragma unroll
    for (int w = 0; w < kHistWarps; ++w) s += sh[w][c];
    if (s) atomicAdd(&hist[c], (unsigned long long)s);
  }
}

cudaError_t launch_hist(const uint8_t* t, uint64_t n, uint64_t* d_hist, int num_sms, cudaStream_t st) {
  cudaError_t err = cudaMemsetAsync(d_hist, 0, 256 * sizeof(uint64_t), st);
  if (err != cudaSuccess) return err;
  if (n == 0) return cudaSuccess;
  const uint64_t vecs = n / 16 + 1;
  const uint64_t per_block = (uint64_t)kHistWarps * 32 * 4;  // aim for >= 4 vectors per thread
  uint64_t want = (vecs + per_block - 1) / per_block;
  uint64_t maxg = (uint64_t)num_sms * 4;
  int grid = (int)(want < 1 ? 1 : (want > maxg ? maxg : want));
  hist_kernel<<<grid, kHistWarps * 32, 0, st>>>(t, n, reinterpret_cast<unsigned long long*>(d_hist));
  return cudaGetLastError();
}

}  // namespace smgpu
