// synth_gen.cu -- device twin of synth.gen_text_host (test/bench input generator).
// Holds no arithmetic of the string-matching method.  Byte i of the text:
//   w = fmix64(key + (i >> 2) * GAMMA);  u16 = (w >> 16*(i & 3)) & 0xFFFF;  t[i] = lut[u16]
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Each thread writes one 8-byte output word covering global bytes [8q, 8q+8) of the
// text (two generator words).  Output buffer starts at global byte `start`.
__global__ void gen_kernel(uint8_t* __restrict__ out, uint64_t start, uint64_t len,
                           uint64_t key, const uint8_t* __restrict__ lut_g) {
  const uint8_t* lut = lut_g;  // 64 KiB, read through the read-only cache
  const uint64_t GAMMA = 0x9E3779B97F4A7C15ull;
  uint64_t q0 = start >> 3, q1 = (start + len + 7) >> 3;
  for (uint64_t q = q0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < q1;
       q += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t wa = fmix64(key + (2 * q) * GAMMA);
    uint64_t wb = fmix64(key + (2 * q + 1) * GAMMA);
    uint8_t b[8];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      b[k] = __ldg(lut + ((wa >> (16 * k)) & 0xFFFF));
      b[4 + k] = __ldg(lut + ((wb >> (16 * k)) & 0xFFFF));
    }
    uint64_t g = q * 8;
    if (g >= start && g + 8 <= start + len && (((uintptr_t)(out + (g - start))) & 7) == 0) {
      uint64_t v = 0;
#pragma unroll
      for (int k = 0; k < 8; k++) v |= (uint64_t)b[k] << (8 * k);
      *reinterpret_cast<uint64_t*>(out + (g - start)) = v;
    } else {
#pragma unroll
      for (int k = 0; k < 8; k++) {
        uint64_t i = g + k;
        if (i >= start && i < start + len) out[i - start] = b[k];
      }
    }
  }
}

}  // namespace

extern "C" int synth_gen_text(void* out, uint64_t start, uint64_t len, uint64_t key,
                              const void* lut_dev, void* stream) {
  if (len == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t words = (len + 16) / 8;
  uint64_t want = (words + 255) / 256;
  int grid = (int)(want < (uint64_t)sms * 4 ? (want ? want : 1) : (uint64_t)sms * 4);
  gen_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((uint8_t*)out, start, len, key,
                                                    (const uint8_t*)lut_dev);
  return (int)cudaGetLastError();
}
