// hist_probe.cu -- byte-histogram kernel variants (A1) for tools/hist_probe.py: per-warp shared
// bins with R lane replicas, W warps per block, U 16-B vectors in flight per thread.
#include <cstdint>
#include <cuda_runtime.h>

template <int W, int R, int U>
__global__ void __launch_bounds__(W * 32) hist_v(const uint4* __restrict__ v, uint64_t nvec,
                                                   unsigned long long* __restrict__ hist) {
  extern __shared__ uint32_t sh[];  // [W][256 * R]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < W * 256 * R; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t* h = sh + warp * 256 * R + (lane % R);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < nvec; i += U * stride) {
    uint4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = __ldcs(v + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t w[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        atomicAdd(&h[(w[k] & 0xFF) * R], 1u);
        atomicAdd(&h[((w[k] >> 8) & 0xFF) * R], 1u);
        atomicAdd(&h[((w[k] >> 16) & 0xFF) * R], 1u);
        atomicAdd(&h[(w[k] >> 24) * R], 1u);
      }
    }
  }
  for (; i < nvec; i += stride) {
    const uint4 a = __ldcs(v + i);
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      atomicAdd(&h[(w[k] & 0xFF) * R], 1u);
      atomicAdd(&h[((w[k] >> 8) & 0xFF) * R], 1u);
      atomicAdd(&h[((w[k] >> 16) & 0xFF) * R], 1u);
      atomicAdd(&h[(w[k] >> 24) * R], 1u);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 256; c += blockDim.x) {
    uint64_t s = 0;
    for (int w = 0; w < W; ++w)
      for (int r = 0; r < R; ++r) s += sh[w * 256 * R + c * R + r];
    if (s) atomicAdd(&hist[c], (unsigned long long)s);
  }
}

// lane-private bins: bins[c][lane] (bank = lane: never a bank conflict, no same-address
// contention), U 16-B vectors in flight per thread, W warps per block
template <int W, int U>
__global__ void __launch_bounds__(W * 32) hist_lp(const uint4* __restrict__ v, uint64_t nvec,
                                                    unsigned long long* __restrict__ hist) {
  extern __shared__ uint32_t sh[];  // [W][256][32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < W * 256 * 32; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t* h = sh + warp * 256 * 32 + lane;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < nvec; i += U * stride) {
    uint4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = __ldcs(v + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t w[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        atomicAdd(&h[(w[k] & 0xFF) * 32], 1u);
        atomicAdd(&h[((w[k] >> 8) & 0xFF) * 32], 1u);
        atomicAdd(&h[((w[k] >> 16) & 0xFF) * 32], 1u);
        atomicAdd(&h[(w[k] >> 24) * 32], 1u);
      }
    }
  }
  for (; i < nvec; i += stride) {
    const uint4 a = __ldcs(v + i);
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      atomicAdd(&h[(w[k] & 0xFF) * 32], 1u);
      atomicAdd(&h[((w[k] >> 8) & 0xFF) * 32], 1u);
      atomicAdd(&h[((w[k] >> 16) & 0xFF) * 32], 1u);
      atomicAdd(&h[(w[k] >> 24) * 32], 1u);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 256; c += blockDim.x) {
    uint64_t s = 0;
    for (int w = 0; w < W; ++w)
      for (int l = 0; l < 32; ++l) s += sh[(w * 256 + c) * 32 + ((l + c) & 31)];
    if (s) atomicAdd(&hist[c], (unsigned long long)s);
  }
}

template <int W, int U>
float run_lp(const void* t, uint64_t n, unsigned long long* d_hist, int bps, int reps) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = (size_t)W * 256 * 32 * 4;
  if (cudaFuncSetAttribute(hist_lp<W, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return -3.f;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t nvec = n / 16;
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaMemsetAsync(d_hist, 0, 256 * 8);
    cudaEventRecord(a);
    hist_lp<W, U><<<sms * bps, W * 32, smem>>>((const uint4*)t, nvec, d_hist);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (cudaGetLastError() != cudaSuccess) return -1.f;
  return (float)(n / (best * 1e-3) / 1e9);
}

template <int W, int R, int U>
float run(const void* t, uint64_t n, unsigned long long* d_hist, int bps, int reps) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = (size_t)W * 256 * R * 4;
  cudaFuncSetAttribute(hist_v<W, R, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t nvec = n / 16;
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaMemsetAsync(d_hist, 0, 256 * 8);
    cudaEventRecord(a);
    hist_v<W, R, U><<<sms * bps, W * 32, smem>>>((const uint4*)t, nvec, d_hist);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (cudaGetLastError() != cudaSuccess) return -1.f;
  return (float)(n / (best * 1e-3) / 1e9);
}

extern "C" float hist_probe(int variant, const void* t, uint64_t n, unsigned long long* d_hist, int bps, int reps) {
  switch (variant) {
    case 0: return run<8, 1, 2>(t, n, d_hist, bps, reps);
    case 1: return run<8, 2, 2>(t, n, d_hist, bps, reps);
    case 2: return run<8, 4, 2>(t, n, d_hist, bps, reps);
    case 3: return run<8, 8, 2>(t, n, d_hist, bps, reps);
    case 4: return run<8, 1, 4>(t, n, d_hist, bps, reps);
    case 5: return run<8, 4, 4>(t, n, d_hist, bps, reps);
    case 6: return run<4, 8, 4>(t, n, d_hist, bps, reps);
    case 7: return run<16, 2, 2>(t, n, d_hist, bps, reps);
    case 8: return run<4, 4, 4>(t, n, d_hist, bps, reps);
    case 9: return run_lp<1, 8>(t, n, d_hist, bps, reps);
    case 10: return run_lp<1, 16>(t, n, d_hist, bps, reps);
    case 11: return run_lp<2, 8>(t, n, d_hist, bps, reps);
    case 12: return run_lp<2, 16>(t, n, d_hist, bps, reps);
    case 13: return run_lp<4, 4>(t, n, d_hist, bps, reps);
    case 14: return run_lp<4, 8>(t, n, d_hist, bps, reps);
    default: return -2.f;
  }
}
