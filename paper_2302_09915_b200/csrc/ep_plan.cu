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
  // every rank's own padded layout: expert segment starts
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    int acc = 0;
    for (int e = 0; e < N; ++e) {
      p.all_lstart[i * N + e] = acc;
      acc += pad16(p.all_counts[i * N + e]);
    }
  }
  if (threadIdx.x == 0) {
    int row = 0;
    for (int el = 0; el < E; ++el) {
      p.seg_start[el] = row;
      for (int i = 0; i < P; ++i) {
        p.src_off[i * E + el] = row;
        row += pad16(p.all_counts[i * N + me * E + el]);
      }
      p.seg_rows[el] = row - p.seg_start[el];
    }
    *p.recv_rows = row;
  }
}

// One warp per receive row: (local expert, source, index) -> the row at the source.
constexpr int kPushWarps = 8;
__global__ void __launch_bounds__(kPushWarps * 32) ep_push_kernel(EpPlanDev p, int P, int E, int me,
                                                                  const __nv_bfloat16* __restrict__ src, PeerBufs dst,
                                                                  int w, int r_max) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * kPushWarps + warp;
  const int total = *p.recv_rows;
  if (r >= total || r >= r_max) return;
  const int N = P * E;
  int el = 0;
  while (el + 1 < E && p.seg_start[el + 1] <= r) ++el;
  int i = 0;
  while (i + 1 < P && p.src_off[(i + 1) * E + el] <= r) ++i;
  const int q = r - p.src_off[i * E + el];
  const int ge = me * E + el;
  if (q >= p.all_counts[i * N + ge]) return;  // padding row
  const long long drow = p.all_lstart[i * N + ge] + q;
  const uint4* s4 = reinterpret_cast<const uint4*>(src + static_cast<long long>(r) * w);
  uint4* d4 = reinterpret_cast<uint4*>(dst.p[i] + drow * w);
  for (int v = lane; v < w / 8; v += 32) d4[v] = s4[v];
}

}  // namespace

void ep_push_back(const EpPlanDev& plan, int P, int E, int me, const __nv_bfloat16* src, const PeerBufs& dst, int w,
                  int r_max, cudaStream_t s) {
  require(w % 8 == 0, "push: row width must be a multiple of 8");
  const int blocks = (r_max + kPushWarps - 1) / kPushWarps;
  ep_push_kernel<<<blocks, kPushWarps * 32, 0, s>>>(plan, P, E, me, src, dst, w, r_max);
  TAMOE_CUDA(cudaGetLastError());
}

void ep_plan_device(const EpPlanDev& plan, int P, int E, int me, cudaStream_t s) {
  require(P >= 1 && P <= kMaxRanks, "expert parallelism supports up to 16 ranks");
  ep_plan_kernel<<<1, 128, 0, s>>>(plan, P, E, me);
  TAMOE_CUDA(cudaGetLastError());
}

}  // namespace tamoe
