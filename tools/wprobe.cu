// Write-bandwidth probe: each warp writes whole regions of `region` 16-B units
// sequentially (region = 0: grid-stride 512-B warp stores, like a fill).
#include <cstdint>
#include <cuda_runtime.h>
__global__ void wkernel(ulonglong2* out, uint64_t n16, uint64_t region) {
  const uint64_t lane = threadIdx.x & 31, gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  if (region == 0) {
    for (uint64_t i = gw * 32 + lane; i < n16; i += nw * 32) out[i] = make_ulonglong2(2 * i, 2 * i + 1);
    return;
  }
  const uint64_t nreg = n16 / region;
  for (uint64_t r = gw; r < nreg; r += nw) {
    ulonglong2* o = out + r * region;
    for (uint64_t i = lane; i < region; i += 32) {
      const uint64_t v = 2 * (r * region + i);
      o[i] = make_ulonglong2(v, v + 1);
    }
  }
}
// 32-B stores per lane (sm_100 256-bit global stores)
__global__ void wkernel32(unsigned long long* out, uint64_t n32, int konst) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid; i < n32; i += nt) {
    const unsigned long long v = konst ? 7ull : 4 * i, d = konst ? 0ull : 1ull;
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(out + 4 * i), "l"(v), "l"(v + d), "l"(v + 2 * d),
                 "l"(v + 3 * d)
                 : "memory");
  }
}
extern "C" float wprobe32(void* p, uint64_t bytes, int blocks_per_sm, int threads, int reps, int konst) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  wkernel32<<<sms * blocks_per_sm, threads>>>((unsigned long long*)p, bytes / 32, konst);
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    wkernel32<<<sms * blocks_per_sm, threads>>>((unsigned long long*)p, bytes / 32, konst);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return (float)(bytes / (best * 1e-3) / 1e9);
}
// non-persistent: each thread writes `per` 16-B units (block-contiguous), then exits
__global__ void wkernel_once(ulonglong2* out, uint64_t n16, int per, int konst) {
  const uint64_t b0 = (uint64_t)blockIdx.x * blockDim.x * per;
  for (int k = 0; k < per; ++k) {
    const uint64_t i = b0 + (uint64_t)k * blockDim.x + threadIdx.x;
    if (i < n16) out[i] = konst ? make_ulonglong2(7, 7) : make_ulonglong2(2 * i, 2 * i + 1);
  }
}
extern "C" float wprobe_once(void* p, uint64_t bytes, int threads, int per, int konst, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t n16 = bytes / 16;
  const uint64_t blocks = (n16 + (uint64_t)threads * per - 1) / ((uint64_t)threads * per);
  wkernel_once<<<(unsigned)blocks, threads>>>((ulonglong2*)p, n16, per, konst);
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    wkernel_once<<<(unsigned)blocks, threads>>>((ulonglong2*)p, n16, per, konst);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return (float)(bytes / (best * 1e-3) / 1e9);
}
// persistent: CTA-contiguous chunks of blockDim x PER units, PER independent stores per thread
template <int PER>
__global__ void wkernel_cta(ulonglong2* out, uint64_t n16) {
  const uint64_t chunk = (uint64_t)blockDim.x * PER, nch = n16 / chunk;
  for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    ulonglong2 v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint64_t i = c * chunk + (uint64_t)k * blockDim.x + threadIdx.x;
      v[k] = make_ulonglong2(2 * i, 2 * i + 1);
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) out[c * chunk + (uint64_t)k * blockDim.x + threadIdx.x] = v[k];
  }
}
extern "C" float wprobe_cta(void* p, uint64_t bytes, int blocks_per_sm, int threads, int per, int reps) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto go = [&] {
    if (per == 4) wkernel_cta<4><<<sms * blocks_per_sm, threads>>>((ulonglong2*)p, bytes / 16);
    else if (per == 8) wkernel_cta<8><<<sms * blocks_per_sm, threads>>>((ulonglong2*)p, bytes / 16);
    else wkernel_cta<1><<<sms * blocks_per_sm, threads>>>((ulonglong2*)p, bytes / 16);
  };
  go();
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    go();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return (float)(bytes / (best * 1e-3) / 1e9);
}
// persistent warps that fetch their next region from an atomic counter (dispatch order
// keeps the write window tight, like the block scheduler does for one-shot grids)
__global__ void wkernel_dyn(ulonglong2* out, uint64_t n16, uint64_t region, unsigned long long* ctr) {
  const int lane = threadIdx.x & 31;
  const uint64_t nreg = n16 / region;
  while (true) {
    unsigned long long r = 0;
    if (lane == 0) r = atomicAdd(ctr, 1ull);
    r = __shfl_sync(0xFFFFFFFFu, r, 0);
    if (r >= nreg) break;
    ulonglong2* o = out + r * region;
    for (uint64_t i = lane; i < region; i += 32) {
      const uint64_t v = 2 * (r * region + i);
      o[i] = make_ulonglong2(v, v + 1);
    }
  }
}
extern "C" float wprobe_dyn(void* p, uint64_t bytes, uint64_t region_bytes, int blocks_per_sm, int threads, int reps) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* ctr;
  cudaMalloc(&ctr, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int i = 0; i <= reps; ++i) {
    cudaMemsetAsync(ctr, 0, 8);
    cudaEventRecord(a);
    wkernel_dyn<<<sms * blocks_per_sm, threads>>>((ulonglong2*)p, bytes / 16, region_bytes / 16, ctr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i && ms < best) best = ms;
  }
  cudaFree(ctr);
  return (float)(bytes / (best * 1e-3) / 1e9);
}
extern "C" float wprobe(void* p, uint64_t bytes, uint64_t region_bytes, int blocks_per_sm, int threads, int reps) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t n16 = bytes / 16, reg = region_bytes / 16;
  wkernel<<<sms * blocks_per_sm, threads>>>((ulonglong2*)p, n16, reg);
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    wkernel<<<sms * blocks_per_sm, threads>>>((ulonglong2*)p, n16, reg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return (float)(bytes / (best * 1e-3) / 1e9);
}
