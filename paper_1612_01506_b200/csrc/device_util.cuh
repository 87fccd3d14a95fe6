// device_util.cuh -- sm_100a primitives used by the string-matching kernels:
// mbarrier ring synchronisation, 1-D TMA bulk copies (cp.async.bulk), L2 cache
// policies, packed-byte (SWAR) equality flags.  Inline PTX, no CUTLASS.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Debug build (-DSMGPU_DEBUG_CHECKS, libsmgpu_debug.so): device-side bounds
// assertions on every global read range and shared-memory window (a stand-in for
// compute-sanitizer, which is not available on this pool).  Compiled out otherwise.
#ifdef SMGPU_DEBUG_CHECKS
#include <cstdio>
#define SMGPU_DCHECK(cond)                                                              \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      printf("SMGPU_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x, #cond);                                 \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define SMGPU_DCHECK(cond) \
  do {                     \
  } while (0)
#endif

namespace smgpu {

// ---------------------------------------------------------------------------
// mbarrier (shared::cta)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t tx) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(bar)),
               "r"(tx)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// for waits that are usually long (the producer waiting for a free stage): let the
// thread be suspended up to `ns` per probe instead of re-issuing the probe
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns = 20000) {
  while (!mbar_try_wait_sleep(bar, parity, ns)) {
  }
}

// generic-proxy writes to smem -> visible to later async-proxy (TMA) writes/reads
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// ---------------------------------------------------------------------------
// NVLink SHARP (NVLS) reduction through a multicast address: the add is applied to the
// bound buffer of every device in the multicast group (PTX multimem.red).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void multimem_red_add_u64(void* mc_addr, unsigned long long v) {
  asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(mc_addr), "l"(v) : "memory");
}

// ---------------------------------------------------------------------------
// global loads
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint8_t ldg_u8_nc(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.global.nc.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<uint8_t>(v);
}

__device__ __forceinline__ uint4 ldg_v4_stream(const void* p, uint64_t policy) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(policy));
  return r;
}

// ---------------------------------------------------------------------------
// shared-memory loads
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 lds128(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }

// ---------------------------------------------------------------------------
// Packed-byte equality (the sm_100a stand-in for SIMDcompare):
// 4 byte lanes per 32-bit register.  bc = symbol * 0x01010101 (the paper's
// "s(y,16)" broadcast).
// ---------------------------------------------------------------------------
// exact: bit 7 of byte k set iff byte k of w == byte k of bc (other bits garbage
// unless masked with 0x80808080)
__device__ __forceinline__ uint32_t eq_flags_raw(uint32_t w, uint32_t bc) {
  uint32_t y = w ^ bc;
  uint32_t t = (y & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;  // bit7 set iff low 7 bits nonzero
  return ~(t | y);                              // bit7 set iff y byte == 0
}
// eq_flags_raw with its add as an IMAD (k1 = 1, opaque to the compiler: a value the caller
// derives from a kernel parameter): the byte compares are ALU-pipe bound, the FMA pipe idles
__device__ __forceinline__ uint32_t eq_flags_fma(uint32_t w, uint32_t bc, uint32_t k1) {
  const uint32_t y = w ^ bc;
  uint32_t t;
  asm("mad.lo.u32 %0, %1, %2, 0x7F7F7F7F;" : "=r"(t) : "r"(y & 0x7F7F7F7Fu), "r"(k1));
  return ~(t | y);
}
// "any byte equal" test term (exact as a whole-word predicate; per-byte bits may
// include false positives above a true match, so it is only ever OR-reduced)
__device__ __forceinline__ uint32_t any_eq_term(uint32_t w, uint32_t bc) {
  uint32_t y = w ^ bc;
  return (y - 0x01010101u) & ~y;
}

// 4-bit mask -> 0x80-per-byte flags
__device__ __forceinline__ uint32_t nibble_to_flags(uint32_t nib) {
  return ((nib * 0x00204081u) & 0x01010101u) << 7;
}

// bytes [s, s+4) of the little-endian pair (lo, hi), s in 0..3 (shift = 8*s)
__device__ __forceinline__ uint32_t byte_window(uint32_t lo, uint32_t hi, uint32_t shift) {
  return __funnelshift_r(lo, hi, shift);
}

}  // namespace smgpu
