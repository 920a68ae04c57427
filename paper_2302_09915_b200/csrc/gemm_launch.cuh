// Host-side launcher of the persistent tcgen05 GEMM engine (one CTA per SM).
#pragma once
#include <algorithm>

#include "common.hpp"
#include "gemm_sm100.cuh"

namespace tamoe {

// kCG = 2 launches CTA pairs (cluster 2x1x1) running tcgen05.mma.cta_group::2 (M = 256 per pair); kCG = 4 two
// pairs per cluster sharing the token operand by TMA multicast (swap GEMMs).
template <int kMode, int BN, bool A_MN, bool B_MN, class Epi, int kCG = 1>
void launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, const typename Epi::Params& ep,
                 int grid_limit, cudaStream_t s) {
  auto kern = gemm_sm100_kernel<kMode, BN, A_MN, B_MN, Epi, kCG>;
  const int smem = GemmSmem<BN, EpiSmem<Epi>::value, kCG>::kTotal;
  static unsigned long long configured = 0;  // per device
  int dev = 0;
  TAMOE_CUDA(cudaGetDevice(&dev));
  if (!((configured >> dev) & 1ull)) {
    TAMOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured |= 1ull << dev;
  }
  int grid = num_sms();
  if (grid_limit > 0 && grid_limit < grid) grid = grid_limit;
  grid = (grid / kCG) * kCG;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if constexpr (kCG > 1) {
    // a persistent grid must be co-resident: GPCs whose SM count is not a multiple of kCG leave SMs idle
    static int max_clusters[64] = {};
    if (max_clusters[dev] == 0) {
      int n = 0;
      cudaLaunchConfig_t occ = cfg;
      occ.numAttrs = 1;  // the cluster shape only
      TAMOE_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &occ));
      max_clusters[dev] = n > 0 ? n : 1;
    }
    grid = std::min(grid, max_clusters[dev] * kCG);
    cfg.gridDim = dim3(grid);
  }
  TAMOE_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, p, ep));
}

}  // namespace tamoe
