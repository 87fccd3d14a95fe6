// search_packed_pre.cu -- NEXT-3: PACKED over a code array packed ONCE per call.
//
// For texts of <= 4 symbols every pattern of a batch compares b-bit codes (reading R20,
// code(x) = (x >> s) & (2^b - 1) injective on the text's symbols).  Instead of packing
// every tile in every pattern's pass, pack_text_kernel converts the text once into a
// code array (1 or 2 bits per byte, base-relative: alignment x <-> bits [b x, b x + b)),
// and each pattern pass TMA-loads the tile's codes (n b / 8 bytes instead of n), with no
// packing and no CTA barrier per tile.  Every alignment is still compared (Alg. 4).
#include "search_dispatch.cuh"

namespace smgpu {
namespace {

// chunk q of the code array = base-relative bytes [16 q, 16 q + 16): bytes outside the
// text t[0..n) (x < delta or x >= delta + n) read as 0 -- their codes are never compared
// for a valid alignment (every compared position lies inside the text)
// support check (bad != nullptr): the code field is injective only on the symbols the
// host chose it for (syms: those four bytes, repeated to fill); a text byte outside
// them sets *bad, and the guarded PACKED launches yield to their byte-compare fallback
__device__ __forceinline__ bool word_in_syms(uint32_t w, uint32_t syms) {
  uint32_t f = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) f |= eq_flags_raw(w, ((syms >> (8 * i)) & 0xFFu) * 0x01010101u);
  return (f & 0x80808080u) == 0x80808080u;
}

template <int B>
__global__ void __launch_bounds__(256) pack_text_kernel(const uint8_t* __restrict__ base, uint64_t delta,
                                                       uint64_t n, uint32_t shift, uint8_t* __restrict__ codes,
                                                       uint64_t nchunks, uint32_t syms, uint32_t* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t lo = delta, hi = delta + n;
  const uint64_t pol = l2_policy_evict_first();
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nchunks; q += stride) {
    const uint64_t x0 = 16u * q;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (x0 >= lo && x0 + 16u <= hi) {
      v = ldg_v4_stream(base + x0, pol);
      if (bad && !(word_in_syms(v.x, syms) && word_in_syms(v.y, syms) && word_in_syms(v.z, syms) &&
                   word_in_syms(v.w, syms)))
        atomicOr(bad, 1u);
    } else if (x0 + 16u > lo && x0 < hi) {
      uint32_t w[4] = {0u, 0u, 0u, 0u};
      bool ok = true;
      for (uint32_t j = 0; j < 16; ++j)
        if (x0 + j >= lo && x0 + j < hi) {
          const uint32_t x = ldg_u8_nc(base + x0 + j);
          w[j >> 2] |= x << (8 * (j & 3));
          ok = ok && word_in_syms(x * 0x01010101u, syms);
        }
      if (bad && !ok) atomicOr(bad, 1u);
      v = make_uint4(w[0], w[1], w[2], w[3]);
    }
    const uint32_t c = pack_chunk<B>(v, shift);
    if (B == 2) reinterpret_cast<uint32_t*>(codes)[q] = c;
    else reinterpret_cast<uint16_t*>(codes)[q] = (uint16_t)c;
  }
}

}  // namespace

cudaError_t launch_search_packed_pre(const HostLaunch& L, cudaStream_t st) {
  if (L.strategy == kPacked2Pre) return launch_strategy<kPacked2Pre>(L, st);
  return launch_strategy<kPacked1Pre>(L, st);
}

cudaError_t launch_pack_text(const uint8_t* base, uint64_t delta, uint64_t n, uint32_t shift, int b, uint8_t* codes,
                             uint64_t code_bytes, uint32_t syms, uint32_t* bad, int num_sms, cudaStream_t st) {
  const uint64_t nchunks = code_bytes / (2u * (uint64_t)b);
  const uint64_t want = (nchunks + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms * 8;
  const int grid = (int)(want < cap ? (want ? want : 1) : cap);
  if (b == 2) pack_text_kernel<2><<<grid, 256, 0, st>>>(base, delta, n, shift, codes, nchunks, syms, bad);
  else pack_text_kernel<1><<<grid, 256, 0, st>>>(base, delta, n, shift, codes, nchunks, syms, bad);
  return cudaGetLastError();
}

}  // namespace smgpu
