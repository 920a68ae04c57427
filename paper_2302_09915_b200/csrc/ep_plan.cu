// Device-side expert-parallel plan from the all-gathered counts (one small CTA; P <= 16, N <= 256).
#include "common.hpp"
#include "ep.hpp"

namespace tamoe {

namespace {

__device__ __forceinline__ int pad16(int c) { return (c + 15) & ~15; }

__global__ void ep_plan_kernel(EpPlanDev p, int P, int E, int me) {
  __shared__ int blk[kMaxRanks * kMaxRanks];  // blk[i*P + j] = padded rows rank i sends to rank j
  const int N = P * E;
  for (int ij = threadIdx.x; ij < P * P; ij += blockDim.x) {
    const int i = ij / P, j = ij % P;
    int r = 0;
    for (int e = 0; e < E; ++e) r += pad16(p.all_counts[i * N + j * E + e]);
    blk[ij] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int recv = 0;
    for (int i = 0; i < P; ++i) {
      int row = recv;
      for (int e = 0; e < E; ++e) {
        const int c = pad16(p.all_counts[i * N + me * E + e]);
        p.seg_start[i * E + e] = row;
        p.seg_rows[i * E + e] = c;
        row += c;
      }
      recv += blk[i * P + me];
    }
    *p.recv_rows = recv;
    int off = 0;
    for (int j = 0; j < P; ++j) {
      int base = 0;
      for (int i = 0; i < me; ++i) base += blk[i * P + j];
      p.dst_base[j] = base;
      p.send_off[j] = off;
      off += blk[me * P + j];
    }
  }
}

}  // namespace

void ep_plan_device(const EpPlanDev& plan, int P, int E, int me, cudaStream_t s) {
  require(P >= 1 && P <= kMaxRanks, "expert parallelism supports up to 16 ranks");
  ep_plan_kernel<<<1, 128, 0, s>>>(plan, P, E, me);
  TAMOE_CUDA(cudaGetLastError());
}

}  // namespace tamoe
