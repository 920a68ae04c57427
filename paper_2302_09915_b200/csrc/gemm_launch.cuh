// Host-side launcher of the persistent tcgen05 GEMM engine (one CTA per SM).
#pragma once
#include "common.hpp"
#include "gemm_sm100.cuh"

namespace tamoe {

template <int kMode, int BN, bool A_MN, bool B_MN, class Epi>
void launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, const typename Epi::Params& ep,
                 int grid_limit, cudaStream_t s) {
  auto kern = gemm_sm100_kernel<kMode, BN, A_MN, B_MN, Epi>;
  const int smem = GemmSmem<BN, EpiSmem<Epi>::value>::kTotal;
  static bool configured = false;
  if (!configured) {
    TAMOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  int grid = num_sms();
  if (grid_limit > 0 && grid_limit < grid) grid = grid_limit;
  kern<<<grid, kGemmThreads, smem, s>>>(ta, tb, p, ep);
  TAMOE_CUDA(cudaGetLastError());
}

}  // namespace tamoe
