// probe.cu -- read-bandwidth probes (measurement infrastructure, not the product):
//   ldg : grid-stride 16-B loads, XOR-reduced (the plain read roof)
//   tma : the search kernel's staging ring (1 producer thread issuing cp.async.bulk
//         into `stages` buffers of `tile` bytes, 8 consumer warps that only wait and
//         release) -- the roof of A3 staging without any compare work.
// Built by tools/probe.py with nvcc -arch sm_100a into tools/libprobe.so.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ldg_kernel(const uint4* __restrict__ p, uint64_t n16, uint32_t* out) {
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride), d = __ldcs(p + i + 3 * stride);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
  }
  for (; i < n16; i += stride) {
    uint4 a = __ldcs(p + i);
    acc ^= a.x ^ a.y ^ a.z ^ a.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// ctr != nullptr: tiles are fetched from that counter by the producer (dynamic dispatch)
// and handed to the consumers through tix[stage]; ~0 ends the ring
__global__ void tma_kernel(const uint8_t* __restrict__ base, uint64_t ntiles, uint32_t tile, uint32_t stages,
                           uint32_t splits, uint32_t* out, unsigned long long* ctr) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 16;
  uint64_t* tix = empty + 16;
  uint8_t* ring = smem + 512;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(nwarps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == nwarps) {
    if (lane != 0) return;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    uint32_t s = 0, ph = 0;
    bool wrapped = false;
    for (uint64_t t0 = blockIdx.x;; t0 += gridDim.x) {
      const uint64_t t = ctr ? atomicAdd(ctr, 1ull) : t0;
      if (wrapped) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0,1,0,p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&empty[s])), "r"(ph ^ 1u), "r"(20000u) : "memory");
      }
      if (t >= ntiles) {
        if (ctr) {
          tix[s] = ~0ull;
          asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(&full[s])) : "memory");
        }
        break;
      }
      tix[s] = t;
      asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                       smem_u32(&full[s])), "r"(tile) : "memory");
      const uint32_t part = tile / splits;
      for (uint32_t k = 0; k < splits; ++k)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                smem_u32(ring + (size_t)s * tile + k * part)),
            "l"(base + t * tile + k * part), "r"(part), "r"(smem_u32(&full[s])), "l"(pol) : "memory");
      if (++s == stages) { s = 0; ph ^= 1u; wrapped = true; }
    }
    return;
  }
  uint32_t s = 0, ph = 0, acc = 0;
  for (uint64_t t = blockIdx.x; ctr || t < ntiles; t += gridDim.x) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&full[s])), "r"(ph) : "memory");
    if (ctr && tix[s] == ~0ull) break;
    acc ^= reinterpret_cast<const uint32_t*>(ring + (size_t)s * tile)[warp * 32 + lane];
    __syncwarp();
    if (lane == 0) asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(&empty[s])) : "memory");
    if (++s == stages) { s = 0; ph ^= 1u; }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

}  // namespace

extern "C" float probe_ldg(const void* p, uint64_t n, int blocks_per_sm, int reps) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint32_t* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t n16 = n / 16;
  ldg_kernel<<<sms * blocks_per_sm, 512>>>((const uint4*)p, n16, out);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) ldg_kernel<<<sms * blocks_per_sm, 512>>>((const uint4*)p, n16, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  return (float)(n16 * 16.0 * reps / (ms * 1e-3) / 1e9);
}

extern "C" float probe_tma(const void* p, uint64_t n, uint32_t tile, uint32_t stages, uint32_t ctas_per_sm,
                           uint32_t splits, int consumer_warps, int reps, int dyn) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  size_t smem = 512 + (size_t)tile * stages;
  unsigned long long* ctr = nullptr;
  if (dyn) {
    cudaMalloc(&ctr, 8 * (reps + 1));
    cudaMemset(ctr, 0, 8 * (reps + 1));
  }
  if (cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return -1.f;
  uint32_t* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t ntiles = n / tile;
  const int threads = (consumer_warps + 1) * 32;
  tma_kernel<<<sms * ctas_per_sm, threads, smem>>>((const uint8_t*)p, ntiles, tile, stages, splits, out, ctr);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r)
    tma_kernel<<<sms * ctas_per_sm, threads, smem>>>((const uint8_t*)p, ntiles, tile, stages, splits, out,
                                                     ctr ? ctr + 1 + r : nullptr);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  cudaFree(out);
  if (ctr) cudaFree(ctr);
  if (e != cudaSuccess) return -2.f;
  return (float)(ntiles * (double)tile * reps / (ms * 1e-3) / 1e9);
}
