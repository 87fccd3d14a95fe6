// param_probe.cu -- host enqueue cost of a kernel launch vs the size of its __grid_constant__ parameter block
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

template <int BYTES>
struct Blk {
  uint32_t w[BYTES / 4];
};
template <int BYTES>
__global__ void k(const __grid_constant__ Blk<BYTES> b, uint32_t* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = b.w[BYTES / 4 - 1];
}
template <int BYTES>
double run(uint32_t* out, int reps) {
  static Blk<BYTES> b;
  std::memset(&b, 1, sizeof(b));
  k<BYTES><<<444, 288>>>(b, out);
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) k<BYTES><<<444, 288>>>(b, out);
  auto t1 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}
int main() {
  uint32_t* out;
  cudaMalloc(&out, 4);
  std::printf("param bytes -> host us per launch (enqueue only, 2000 launches)\n");
  std::printf("%6d %8.2f\n", 256, run<256>(out, 2000));
  std::printf("%6d %8.2f\n", 4096, run<4096>(out, 2000));
  std::printf("%6d %8.2f\n", 8192, run<8192>(out, 2000));
  std::printf("%6d %8.2f\n", 12288, run<12288>(out, 2000));
  std::printf("%6d %8.2f\n", 16384, run<16384>(out, 2000));
  std::printf("%6d %8.2f\n", 24576, run<24576>(out, 2000));
  std::printf("%6d %8.2f\n", 32000, run<32000>(out, 2000));
  return 0;
}
