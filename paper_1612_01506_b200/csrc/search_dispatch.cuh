// search_dispatch.cuh -- host-side dispatch over the kernel's template parameters
// for ONE strategy (included by search_filter.cu / search_block.cu so the two
// strategies compile in parallel).
#pragma once
#include <cstring>

#include "search_impl.cuh"

namespace smgpu {
namespace {

template <int STRAT, int EPI, int CAP, int CPL>
cudaError_t launch_one(const HostLaunch& L, cudaStream_t st) {
  auto kfn = search_kernel<STRAT, EPI, CAP, CPL>;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  // the attribute belongs to the device's context: set once per (kernel, device)
  static bool attr_done[64] = {};  // benign race: idempotent attribute set
  if (!attr_done[dev]) {
    cudaError_t err = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (err != cudaSuccess) return err;
    attr_done[dev] = true;
  }
  // persistent grid: never more CTAs than can be resident at once (registers or shared
  // memory may allow fewer per SM than the host's plan assumed) -- a second wave of CTAs
  // would run the round-robin work items after the first, a tail of up to 50 %
  int grid = L.grid;
  {
    static thread_local size_t cached_smem = ~(size_t)0;
    static thread_local int cached_dev = -1;
    static thread_local int cached_blocks = 0;
    if (cached_smem != L.smem || cached_dev != dev) {
      int nb = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kfn, kThreads, L.smem) != cudaSuccess) nb = 0;
      cached_smem = L.smem;
      cached_dev = dev;
      cached_blocks = nb;
    }
    int sms = 0;
    if (cached_blocks > 0 &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
      grid = grid < cached_blocks * sms ? grid : cached_blocks * sms;
  }
  static thread_local LaunchParams<CAP> P;  // ~19 KiB for CAP = 4096: keep it off the stack
  P.a = L.a;
  std::memset(P.d, 0, sizeof(P.d));
  std::memcpy(P.d, L.d.data(), L.d.size() * sizeof(PatDesc));
  std::memcpy(P.e, L.e.data(), L.e.size() * sizeof(uint32_t));
  kfn<<<grid, kThreads, L.smem, st>>>(P);
  return cudaGetLastError();
}

template <int STRAT, int EPI, int CPL>
cudaError_t launch_cap(const HostLaunch& L, cudaStream_t st) {
  if (L.e.size() <= (size_t)kTableSmall) return launch_one<STRAT, EPI, kTableSmall, CPL>(L, st);
  if (L.e.size() <= (size_t)kTableMid) return launch_one<STRAT, EPI, kTableMid, CPL>(L, st);
  return launch_one<STRAT, EPI, kTableLarge, CPL>(L, st);
}

template <int STRAT, int EPI>
cudaError_t launch_c(const HostLaunch& L, cudaStream_t st) {
  switch (L.cpl) {
    case 8: return launch_cap<STRAT, EPI, 8>(L, st);
    case 4: return launch_cap<STRAT, EPI, 4>(L, st);
    case 2: return launch_cap<STRAT, EPI, 2>(L, st);
    default: return launch_cap<STRAT, EPI, 1>(L, st);
  }
}

// NEXT-4 count launches with the multicast epilogue: large tables only (fewer instantiations)
template <int STRAT>
cudaError_t launch_mc(const HostLaunch& L, cudaStream_t st) {
  switch (L.cpl) {
    case 8: return launch_one<STRAT, kEpiCountMc, kTableLarge, 8>(L, st);
    case 4: return launch_one<STRAT, kEpiCountMc, kTableLarge, 4>(L, st);
    case 2: return launch_one<STRAT, kEpiCountMc, kTableLarge, 2>(L, st);
    default: return launch_one<STRAT, kEpiCountMc, kTableLarge, 1>(L, st);
  }
}

template <int STRAT>
cudaError_t launch_strategy(const HostLaunch& L, cudaStream_t st) {
  if (L.epilogue == kEpiCount) return launch_c<STRAT, kEpiCount>(L, st);
  if (L.epilogue == kEpiCountMc) return launch_mc<STRAT>(L, st);
  if (L.epilogue == kEpiStage) return launch_c<STRAT, kEpiStage>(L, st);
  return launch_c<STRAT, kEpiWrite>(L, st);
}

}  // namespace
}  // namespace smgpu
