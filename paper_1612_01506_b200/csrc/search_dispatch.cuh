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
    // occupancy per (device, dynamic smem): the launches of one batch call differ in their
    // stage size, so a few entries (round-robin replacement) keep the occupancy query, a
    // few microseconds of host time, off every launch
    struct OccEntry {
      size_t smem;
      int dev, blocks, sms;
    };
    constexpr int kOccEntries = 8;
    static thread_local OccEntry occ[kOccEntries] = {};
    static thread_local int occ_used = 0, occ_next = 0;
    int hit = -1;
    for (int i = 0; i < occ_used; ++i)
      if (occ[i].smem == L.smem && occ[i].dev == dev) {
        hit = i;
        break;
      }
    if (hit < 0) {
      OccEntry x{L.smem, dev, 0, 0};
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x.blocks, kfn, kThreads, L.smem) != cudaSuccess) x.blocks = 0;
      if (cudaDeviceGetAttribute(&x.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) x.sms = 0;
      cudaGetLastError();  // a failed query only leaves the grid as planned
      hit = occ_used < kOccEntries ? occ_used++ : occ_next++ % kOccEntries;
      occ[hit] = x;
    }
    const OccEntry& o = occ[hit];
    if (o.blocks > 0 && o.sms > 0) grid = grid < o.blocks * o.sms ? grid : o.blocks * o.sms;
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
