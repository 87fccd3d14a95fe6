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
  static bool attr_done = false;  // benign race: idempotent attribute set
  if (!attr_done) {
    cudaError_t err = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (err != cudaSuccess) return err;
    attr_done = true;
  }
  static thread_local LaunchParams<CAP> P;  // ~19 KiB for CAP = 4096: keep it off the stack
  P.a = L.a;
  std::memset(P.d, 0, sizeof(P.d));
  std::memcpy(P.d, L.d.data(), L.d.size() * sizeof(PatDesc));
  std::memcpy(P.e, L.e.data(), L.e.size() * sizeof(uint32_t));
  kfn<<<L.grid, kThreads, L.smem, st>>>(P);
  return cudaGetLastError();
}

template <int STRAT, int EPI, int CPL>
cudaError_t launch_cap(const HostLaunch& L, cudaStream_t st) {
  if (L.e.size() <= (size_t)kTableSmall) return launch_one<STRAT, EPI, kTableSmall, CPL>(L, st);
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

template <int STRAT>
cudaError_t launch_strategy(const HostLaunch& L, cudaStream_t st) {
  if (L.epilogue == kEpiCount) return launch_c<STRAT, kEpiCount>(L, st);
  if (L.epilogue == kEpiStage) return launch_c<STRAT, kEpiStage>(L, st);
  return launch_c<STRAT, kEpiWrite>(L, st);
}

}  // namespace
}  // namespace smgpu
