// alu_probe.cu -- INT-ALU pipe and issue ceilings of one B200,
// the peaks the compare-bound strategies (PACKED on sigma <= 4 texts, periodic text)
// are measured against.  Each thread runs kChains independent dependent chains of
// LOP3 or SHF (ALU-pipe instructions, SASS-checked by tools/alu_probe.py),
// so the ALU pipe, not latency, is the limit.  Grid = SMs x blocks_per_sm, 256 threads.
#include <cstdint>
#include <cuda_runtime.h>

namespace {
constexpr int kChains = 8;

template <int OP>
__global__ void __launch_bounds__(256) alu_kernel(uint32_t* out, uint32_t iters, uint32_t seed) {
  uint32_t x[kChains], y = seed ^ threadIdx.x, z = seed * 0x9E3779B9u + blockIdx.x;
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = seed + c * 0x01010101u + threadIdx.x;
  for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (OP == 0) {  // LOP3: x = (x ^ y) & ~z | ...  one LOP3 each
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
        } else if (OP == 1) {  // SHF (funnel shift, the PACKED step's window extraction)
          asm volatile("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
        } else {  // IADD3
          asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(y));
        }
      }
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) r ^= x[c];
  if (r == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = r;  // keep the chains alive
}
}  // namespace

extern "C" {
// returns ms of one launch (best of reps); ops = threads * iters * kChains * 4 instructions
float alu_probe(int op, int blocks, uint32_t iters, int reps) {
  uint32_t* out = nullptr;
  cudaMalloc(&out, (size_t)blocks * 256 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < reps + 1; ++r) {
    cudaEventRecord(a);
    if (op == 0) alu_kernel<0><<<blocks, 256>>>(out, iters, 7u + r);
    else if (op == 1) alu_kernel<1><<<blocks, 256>>>(out, iters, 7u + r);
    else alu_kernel<2><<<blocks, 256>>>(out, iters, 7u + r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;  // first launch is warm-up
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  return best;
}
int alu_probe_ops_per_iter() { return kChains * 4; }
}
