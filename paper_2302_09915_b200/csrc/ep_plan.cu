// Device-side expert-parallel plan from the all-gathered counts (one small CTA; P <= 16, N <= 256).
#include "common.hpp"
#include "ep.hpp"

namespace tamoe {

namespace {

__device__ __forceinline__ int pad16(int c) { return (c + 15) & ~15; }

// expert-major receive layouts: at rank j, local expert e_l owns rows
//   [ sum_{e' < e_l} sum_src pad16(c[src][jE+e']) , ... ) split into per-source segments in rank order.
__global__ void ep_plan_kernel(EpPlanDev p, int P, int E, int me) {
  const int N = P * E;
  // one thread per global expert: where do my rows for it start at its owner?
  for (int ge = threadIdx.x; ge < N; ge += blockDim.x) {
    const int j = ge / E, el = ge % E;
    int off = 0;
    for (int e2 = 0; e2 < el; ++e2)
      for (int i = 0; i < P; ++i) off += pad16(p.all_counts[i * N + j * E + e2]);
    for (int i = 0; i < me; ++i) off += pad16(p.all_counts[i * N + ge]);
    p.dst_off[ge] = off;
  }
  if (threadIdx.x == 0) {
    int row = 0;
    for (int el = 0; el < E; ++el) {
      p.seg_start[el] = row;
      for (int i = 0; i < P; ++i) row += pad16(p.all_counts[i * N + me * E + el]);
      p.seg_rows[el] = row - p.seg_start[el];
    }
    *p.recv_rows = row;
  }
}

}  // namespace

void ep_plan_device(const EpPlanDev& plan, int P, int E, int me, cudaStream_t s) {
  require(P >= 1 && P <= kMaxRanks, "expert parallelism supports up to 16 ranks");
  ep_plan_kernel<<<1, 128, 0, s>>>(plan, P, E, me);
  TAMOE_CUDA(cudaGetLastError());
}

}  // namespace tamoe
