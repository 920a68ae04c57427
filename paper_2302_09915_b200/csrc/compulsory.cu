// Compulsory-quota routing (FasterMoE-style ablation, trainer.cpp:121-169): per process,
// tokens in (top-1 score desc, token asc) order each claim their most probable expert (probability desc,
// expert asc) that still has quota; quota_i = LRR(c_hat_i / sum(c_hat_i) * S, S).  Top-1 only; every
// token ends up kept.
//
// Device plan: a stable descending segmented radix sort of the top-1 scores gives the claim order (ties
// keep token order); one warp per process then walks it sequentially (the claims depend on each other),
// each claim a masked warp arg-max over the token's fp64 probabilities with the next token's row already
// loaded; the 32-token expert histograms are rebuilt for the bucket pass that follows.
#include <cub/cub.cuh>

#include "common.hpp"
#include "route.hpp"

namespace tamoe {

namespace {

__global__ void claim_order_init(int* tok, int* offsets, int P, int S) {
  const long long n = static_cast<long long>(P) * S;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    tok[i] = static_cast<int>(i % S);
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i <= P; i += blockDim.x) offsets[i] = i * S;
}

template <int EPL>
__global__ void __launch_bounds__(32) claim_kernel(RouteDims d, RouteBuffers b, const double* __restrict__ probs,
                                                   const int* __restrict__ quota, const int* __restrict__ order) {
  constexpr int NC = EPL * 32;
  __shared__ int q[NC];
  const int proc = blockIdx.x, lane = threadIdx.x;
  const int N = d.N, S = d.S;
  for (int e = lane; e < NC; e += 32) q[e] = e < N ? quota[proc * N + e] : 0;
  __syncwarp();
  const int* ord = order + static_cast<long long>(proc) * S;
  double p[EPL], pn[EPL];
  auto load = [&](int r, double (&dst)[EPL]) {
    const long long g = static_cast<long long>(proc) * S + ord[r];
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int c = j * 32 + lane;
      dst[j] = c < N ? probs[g * N + c] : -1.0;
    }
  };
  if (S > 0) load(0, p);
  for (int r = 0; r < S; ++r) {
    if (r + 1 < S) load(r + 1, pn);
    double bp = -2.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int c = j * 32 + lane;
      if (c < N && q[c] > 0 && p[j] > bp) {
        bp = p[j];
        bi = c;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double op = __shfl_xor_sync(0xffffffffu, bp, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (op > bp || (op == bp && oi < bi)) {
        bp = op;
        bi = oi;
      }
    }
    if (lane == 0) {
      const long long g = static_cast<long long>(proc) * S + ord[r];
      if (bi < N) {  // sum(quota) == S: every token finds a slot
        q[bi] -= 1;
        b.idx[g] = bi;
        b.score[g] = bp;
        b.gate[g] = static_cast<float>(bp);
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < EPL; ++j) p[j] = pn[j];
  }
}

// hist4[group][e] = tokens of the 32-token group routed to e (k = 1), the layout route_bucket consumes
__global__ void __launch_bounds__(32) rebuild_hist_kernel(RouteDims d, RouteBuffers b) {
  const int g = blockIdx.x, lane = threadIdx.x;
  const int groups = d.TB * 4;
  const int proc = g / groups;
  const int tok = (g % groups) * 32 + lane;
  const bool valid = tok < d.S;
  const int e_mine = valid ? b.idx[static_cast<long long>(proc) * d.S + tok] : -1;
  for (int e = 0; e < d.N; ++e) {
    const unsigned bal = __ballot_sync(0xffffffffu, e_mine == e);
    if (lane == 0) b.hist4[static_cast<long long>(g) * d.N + e] = __popc(bal);
  }
}

}  // namespace

size_t compulsory_workspace_bytes(int P, int S) {
  const long long n = static_cast<long long>(P) * S;
  size_t temp = 0;
  cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, temp, static_cast<const double*>(nullptr),
                                                     static_cast<double*>(nullptr), static_cast<const int*>(nullptr),
                                                     static_cast<int*>(nullptr), static_cast<int>(n), P,
                                                     static_cast<const int*>(nullptr), static_cast<const int*>(nullptr));
  auto al = [](size_t v) { return (v + 255) & ~static_cast<size_t>(255); };
  return al(temp) + al(sizeof(double) * n) + 2 * al(sizeof(int) * n) + al(sizeof(int) * (P + 1));
}

void route_compulsory(const RouteDims& d, const RouteBuffers& b, const double* probs, const int* quota, void* ws,
                      size_t ws_bytes, cudaStream_t s) {
  require(d.k == 1, "compulsory routing supports top-1 only");
  require(d.N <= 256, "compulsory routing: N must be <= 256");
  const long long n = static_cast<long long>(d.P) * d.S;
  auto al = [](size_t v) { return (v + 255) & ~static_cast<size_t>(255); };
  size_t temp = 0;
  cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, temp, static_cast<const double*>(nullptr),
                                                     static_cast<double*>(nullptr), static_cast<const int*>(nullptr),
                                                     static_cast<int*>(nullptr), static_cast<int>(n), d.P,
                                                     static_cast<const int*>(nullptr), static_cast<const int*>(nullptr));
  require(ws_bytes >= compulsory_workspace_bytes(d.P, d.S), "compulsory routing: workspace too small");
  char* w = static_cast<char*>(ws);
  void* tmp = w;
  w += al(temp);
  double* keys_out = reinterpret_cast<double*>(w);
  w += al(sizeof(double) * n);
  int* tok_in = reinterpret_cast<int*>(w);
  w += al(sizeof(int) * n);
  int* tok_out = reinterpret_cast<int*>(w);
  w += al(sizeof(int) * n);
  int* offsets = reinterpret_cast<int*>(w);
  claim_order_init<<<static_cast<unsigned>(std::min<long long>((n + 255) / 256, 1024)), 256, 0, s>>>(tok_in, offsets,
                                                                                                     d.P, d.S);
  TAMOE_CUDA(cudaGetLastError());
  // stable radix sort: equal scores keep ascending token order (trainer.cpp:141-146)
  TAMOE_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(tmp, temp, b.score, keys_out, tok_in, tok_out,
                                                                static_cast<int>(n), d.P, offsets, offsets + 1, 0, 64,
                                                                s));
  if (d.N <= 32) claim_kernel<1><<<d.P, 32, 0, s>>>(d, b, probs, quota, tok_out);
  else if (d.N <= 64) claim_kernel<2><<<d.P, 32, 0, s>>>(d, b, probs, quota, tok_out);
  else if (d.N <= 128) claim_kernel<4><<<d.P, 32, 0, s>>>(d, b, probs, quota, tok_out);
  else claim_kernel<8><<<d.P, 32, 0, s>>>(d, b, probs, quota, tok_out);
  TAMOE_CUDA(cudaGetLastError());
  rebuild_hist_kernel<<<static_cast<unsigned>(d.tiles()) * 4, 32, 0, s>>>(d, b);
  TAMOE_CUDA(cudaGetLastError());
}

}  // namespace tamoe
