// search_dispatch.cuh -- host-side dispatch over the kernel's template parameters
// for ONE strategy (included by search_filter.cu / search_block.cu so the two
// strategies compile in parallel).
#pragma once
#include "search_impl.cuh"

namespace smgpu {
namespace {

template <int STRAT, int EPI, int MAXM, int CPL>
cudaError_t launch_one(const SearchArgs& a, const uint32_t* e, uint32_t m, int grid, size_t smem,
                       cudaStream_t st) {
  auto kfn = search_kernel<STRAT, EPI, MAXM, CPL>;
  static bool attr_done = false;  // benign race: idempotent attribute set
  if (!attr_done) {
    cudaError_t err = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (err != cudaSuccess) return err;
    attr_done = true;
  }
  PatternTable<MAXM> pt;
  for (uint32_t q = 0; q < m; ++q) pt.e[q] = e[q];
  for (uint32_t q = m; q < (uint32_t)MAXM; ++q) pt.e[q] = 0;
  kfn<<<grid, kThreads, smem, st>>>(a, pt);
  return cudaGetLastError();
}

template <int STRAT, int EPI, int CPL>
cudaError_t launch_m(const SearchArgs& a, const uint32_t* e, uint32_t m, int grid, size_t smem, cudaStream_t st) {
  if (m <= 64) return launch_one<STRAT, EPI, 64, CPL>(a, e, m, grid, smem, st);
  if (m <= 1024) return launch_one<STRAT, EPI, 1024, CPL>(a, e, m, grid, smem, st);
  return launch_one<STRAT, EPI, 4096, CPL>(a, e, m, grid, smem, st);
}

template <int STRAT, int EPI>
cudaError_t launch_c(const SearchArgs& a, const uint32_t* e, uint32_t m, int cpl, int grid, size_t smem,
                     cudaStream_t st) {
  switch (cpl) {
    case 8: return launch_m<STRAT, EPI, 8>(a, e, m, grid, smem, st);
    case 4: return launch_m<STRAT, EPI, 4>(a, e, m, grid, smem, st);
    case 2: return launch_m<STRAT, EPI, 2>(a, e, m, grid, smem, st);
    default: return launch_m<STRAT, EPI, 1>(a, e, m, grid, smem, st);
  }
}

template <int STRAT>
cudaError_t launch_strategy(const SearchArgs& a, const uint32_t* e, int epi, int cpl, int grid, size_t smem,
                            cudaStream_t st) {
  if (epi == kEpiCount) return launch_c<STRAT, kEpiCount>(a, e, a.m, cpl, grid, smem, st);
  if (epi == kEpiTileCount) return launch_c<STRAT, kEpiTileCount>(a, e, a.m, cpl, grid, smem, st);
  return launch_c<STRAT, kEpiWrite>(a, e, a.m, cpl, grid, smem, st);
}

}  // namespace
}  // namespace smgpu
