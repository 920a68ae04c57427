// Gate: logits = x . Wg^T on tcgen05 (TMA-staged, fp32 accumulate in TMEM,
// fp32 logits out of the epilogue), then a warp-per-8-tokens router: fp64
// softmax exactly as the reference (max-subtract, exp, sequential sum over
// experts, divide: gate.cpp:12-28), top-k (gate.cpp:117-134), per-group
// expert histograms and probability partial sums for the aux loss
// (gate.cpp:115).
//
// Replaces gate_forward (gate.cpp:30-32) + the per-token part of topk_route.
#include <cuda_bf16.h>

#include <cmath>

#include "common.hpp"
#include "gate.hpp"
#include "gemm_launch.cuh"
#include "route_row.cuh"
#include "tma_host.hpp"

namespace tamoe {

struct GateEpiParams {
  float* logits;  // [P*S x N] fp32
  int N, S;
};

// The gate GEMM's epilogue only materialises the fp32 logits (4 B x N per token, L2-resident for the router
// that follows); the two warps of a TMEM lane quarter split the 32-column chunks.
struct EpiLogits {
  using Params = GateEpiParams;
  static constexpr bool kEarlyRelease = true;
  static __device__ __forceinline__ void finish(const Params&, int) {}
  static __device__ __forceinline__ void prefetch(const Params&, const GemmParams&, const TileInfo&, int, int, int,
                                                  uint8_t*, const int*) {}
  template <class Release>
  static __device__ __forceinline__ void run(const Params& e, const GemmParams&, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int h, int lane, uint8_t*, const int*,
                                             Release&& release) {
    const int tok = ti.m0 + q * 32 + lane;
    const bool valid = tok < e.S;
    const long long gtok = static_cast<long long>(ti.g) * e.S + tok;
    const int N = e.N;
    const int C = (N + 31) / 32, C0 = (C + 1) / 2;
    const int cb = h == 0 ? 0 : C0, ce = h == 0 ? C0 : C;
    for (int ch = cb; ch < ce; ++ch) {
      const int c0 = ch * 32;
      float v[32];
      load_acc32(tmem_tile, c0, v);
      if (ch + 1 == ce) release();
      if (!valid) continue;
      float* dst = e.logits + gtok * N + c0;
      if (c0 + 32 <= N && (N % 4) == 0) {
#pragma unroll
        for (int c = 0; c < 32; c += 4) *reinterpret_cast<float4*>(dst + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c0 + c < N) dst[c] = v[c];
      }
    }
    if (cb >= ce) release();
  }
};

// Per-token routing over fp32 logits: fp64 softmax exactly as the reference (max-subtract, exp, sequential
// sum in expert order, divide: gate.cpp:12-28), top-k in (probability desc, expert asc) order
// (gate.cpp:117-134), per-32-token-group expert histograms and probability sums (gate.cpp:115).
// A block of 16 warps owns one 32-token group (= one hist4/msum4 slot); each warp takes 2 tokens with its
// lanes across experts (expert c on lane c % 32), so every exp is computed once and parked in shared
// memory for the sequential denominator, and top-k is a warp arg-max.  (2 tokens per warp: the per-warp
// chain of dependent loads, shuffles and the serial fp64 denominator is the kernel's critical path.)
constexpr int kRouteRowsPerWarp = 2;
constexpr int kRouteGroupWarps = 32 / kRouteRowsPerWarp;

template <int EPL, int KM>
__global__ void __launch_bounds__(kRouteGroupWarps * 32) route_logits_kernel(const float* __restrict__ logits, RouteDims d,
                                                           RowRouteOut o) {
  constexpr int NC = EPL * 32;
  constexpr int RPW = kRouteRowsPerWarp;
  extern __shared__ double route_smem[];
  constexpr int WPG = kRouteGroupWarps;
  auto E = reinterpret_cast<double (*)[RPW][NC + 1]>(route_smem);  // [WPG][RPW][NC+1] exps
  __shared__ double den[WPG][RPW];
  auto ms = reinterpret_cast<double (*)[NC]>(route_smem);            // reuses E after the block barrier
  auto hs = reinterpret_cast<int (*)[NC]>(route_smem + WPG * NC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x;  // 32-token group == hist4 / msum4 slot
  const int groups = d.TB * 4;
  const int proc = b / groups;
  const int tok0 = (b % groups) * 32 + warp * RPW;
  const int N = d.N, k = d.k;
  // rows with a non-finite logit (the reference throws ValidationError, gate.cpp:16-17): the bad flag is
  // raised and the row is routed to experts 0..k-1 with NaN gate values, so every index stays in range and
  // the step's outputs and losses come out NaN (poisoned) instead of faulting on a garbage index
  unsigned okmask = 0;
#pragma unroll 2
  for (int r = 0; r < RPW; ++r) {
    const int tok = tok0 + r;
    const bool valid = tok < d.S;
    const float* row = logits + (static_cast<long long>(proc) * d.S + tok) * N;
    float v[EPL];
    float mx = -INFINITY;
    bool finite = true;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int c = j * 32 + lane;
      v[j] = (valid && c < N) ? __ldg(row + c) : -INFINITY;
      if (valid && c < N) finite &= isfinite(v[j]);
      mx = fmaxf(mx, v[j]);
    }
    if (__all_sync(0xffffffffu, finite)) okmask |= 1u << r;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const double dmx = valid ? static_cast<double>(mx) : 0.0;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int c = j * 32 + lane;
      E[warp][r][c] = (valid && c < N) ? exp(static_cast<double>(v[j]) - dmx) : 0.0;
    }
  }
  __syncwarp();
  if (lane < RPW) {  // sequential denominator, expert order (gate.cpp:19-21)
    double sum = 0.0;
    for (int c = 0; c < N; ++c) sum += E[warp][lane][c];
    den[warp][lane] = sum;
  }
  __syncwarp();
  int hc[EPL];
  double msum[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    hc[j] = 0;
    msum[j] = 0.0;
  }
  for (int r = 0; r < RPW; ++r) {
    const int tok = tok0 + r;
    const bool valid = tok < d.S;
    const long long gtok = static_cast<long long>(proc) * d.S + tok;
    const double dn = den[warp][r];
    const bool ok = (okmask >> r) & 1u;
    double p[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int c = j * 32 + lane;
      p[j] = (valid && c < N) ? (ok ? E[warp][r][c] / dn : __longlong_as_double(0x7ff8000000000000ll)) : 0.0;
      if (valid && c < N && o.probs) o.probs[gtok * N + c] = p[j];
      msum[j] += p[j];
      if (!ok) p[j] = -static_cast<double>(c) / 2048.0;  // selection order of a bad row: experts 0, 1, ...
    }
    if (!valid) continue;
    // top-k: k rounds of a warp arg-max under (p desc, expert asc)
    unsigned taken = 0;
    double pp[KM];
    int pe[KM];
#pragma unroll
    for (int t = 0; t < KM; ++t) {
      pp[t] = -1.0;
      pe[t] = -1;
      if (t < k) {
        double bp = -1.0;
        int bi = 0x7fffffff;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const int c = j * 32 + lane;
          if (c < N && !((taken >> j) & 1u) && p[j] > bp) {
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
        pp[t] = bp;
        pe[t] = bi;
        if ((bi & 31) == lane) {
          taken |= 1u << (bi >> 5);
#pragma unroll
          for (int j = 0; j < EPL; ++j)
            if (j == (bi >> 5)) ++hc[j];
        }
      }
    }
    if (lane == 0) {
      double mass = 0.0;
#pragma unroll
      for (int t = 0; t < KM; ++t)
        if (t < k) mass += pp[t];
#pragma unroll
      for (int t = 0; t < KM; ++t) {
        if (t < k) {
          const long long a = gtok * k + t;
          o.idx[a] = pe[t];
          o.score[a] = ok ? pp[t] : 0.0;
          const double g = !ok ? __longlong_as_double(0x7ff8000000000000ll) : (k == 1 ? pp[t] : pp[t] / mass);
          o.gate[a] = static_cast<float>(g);
          if (o.gate64) o.gate64[a] = g;
        }
      }
    }
  }
  if (okmask != (1u << RPW) - 1u && lane == 0) {
    bool any_bad = false;
    for (int r = 0; r < RPW; ++r) any_bad |= !((okmask >> r) & 1u) && tok0 + r < d.S;
    if (any_bad) atomicOr(o.bad, 1);
  }
  __syncthreads();  // every warp is done with E
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    hs[warp][j * 32 + lane] = hc[j];
    ms[warp][j * 32 + lane] = msum[j];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < N; c += blockDim.x) {
    int hsum = 0;
    double msum_c = 0.0;
#pragma unroll
    for (int w = 0; w < WPG; ++w) {  // fixed order: deterministic
      hsum += hs[w][c];
      msum_c += ms[w][c];
    }
    o.hist4[static_cast<long long>(b) * N + c] = hsum;
    o.msum4[static_cast<long long>(b) * N + c] = msum_c;
  }
}

template <int EPL, int KM>
static void route_logits_launch_k(const float* logits, const RouteDims& d, const RowRouteOut& o, cudaStream_t s) {
  constexpr int smem = kRouteGroupWarps * kRouteRowsPerWarp * (EPL * 32 + 1) * 8;
  static_assert(smem >= kRouteGroupWarps * EPL * 32 * 12, "E must cover the reduction scratch");
  static unsigned long long attr_set = 0;  // per device
  int dev = 0;
  TAMOE_CUDA(cudaGetDevice(&dev));
  if (!((attr_set >> dev) & 1ull)) {
    TAMOE_CUDA(cudaFuncSetAttribute(route_logits_kernel<EPL, KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set |= 1ull << dev;
  }
  route_logits_kernel<EPL, KM><<<static_cast<unsigned>(d.tiles()) * 4, kRouteGroupWarps * 32, smem, s>>>(logits, d, o);
  TAMOE_CUDA(cudaGetLastError());
}

template <int EPL>
static void route_logits_launch(const float* logits, const RouteDims& d, const RowRouteOut& o, cudaStream_t s) {
  if (d.k == 1) route_logits_launch_k<EPL, 1>(logits, d, o, s);
  else if (d.k == 2) route_logits_launch_k<EPL, 2>(logits, d, o, s);
  else route_logits_launch_k<EPL, kMaxTopK>(logits, d, o, s);
}

void route_from_logits(const float* logits, const RouteDims& d, const RowRouteOut& o, cudaStream_t s) {
  require(d.k >= 1 && d.k <= kMaxTopK && d.k <= d.N, "k must be in [1, min(N, 8)]");
  require(d.N <= 256, "router: N must be <= 256");
  if (d.N <= 32) route_logits_launch<1>(logits, d, o, s);
  else if (d.N <= 64) route_logits_launch<2>(logits, d, o, s);
  else if (d.N <= 128) route_logits_launch<4>(logits, d, o, s);
  else route_logits_launch<8>(logits, d, o, s);
}

// Standalone router over caller-provided fp64 probabilities (the reference's topk_route input).
__global__ void __launch_bounds__(kRouteTile) route_rows_kernel(const double* __restrict__ probs, RouteDims d,
                                                               RowRouteOut o) {
  const int tile = blockIdx.x;
  const int proc = tile / d.TB;
  const int tok = (tile % d.TB) * kRouteTile + threadIdx.x;
  const bool valid = tok < d.S;
  const long long gtok = static_cast<long long>(proc) * d.S + tok;
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile_warp = tile * 4 + q;
  TopK<kMaxTopK> tk;
  tk.init();
  double* msum = o.msum4 + static_cast<long long>(tile_warp) * d.N;
  const double* row = probs + gtok * d.N;
  for (int e = 0; e < d.N; ++e) {
    const double pr = valid ? row[e] : 0.0;
    tk.insert(pr, e, d.k);
    const double s = warp_sum_f64(pr);
    if (lane == 0) msum[e] = s;
  }
  finish_row(tk, valid, gtok, d.k, d.N, tile_warp, o, lane);
}

void route_rows_from_probs(const double* probs, const RouteDims& d, const RowRouteOut& o, cudaStream_t s) {
  require(d.k >= 1 && d.k <= kMaxTopK && d.k <= d.N, "k must be in [1, min(N, 8)]");
  route_rows_kernel<<<d.tiles(), kRouteTile, 0, s>>>(probs, d, o);
  TAMOE_CUDA(cudaGetLastError());
}

void gate_forward(const __nv_bfloat16* x, const __nv_bfloat16* wg, int n_pad, const RouteDims& d, int dm,
                  const RowRouteOut& o, cudaStream_t s) {
  require(d.k >= 1 && d.k <= kMaxTopK && d.k <= d.N, "k must be in [1, min(N, 8)]");
  require(dm % 64 == 0, "gate: d must be a multiple of 64 (pad with zeros)");
  require(n_pad % 16 == 0 && n_pad >= d.N && n_pad <= 256, "gate: n_pad must be round_up(N, 16) <= 256");
  require(o.logits != nullptr, "gate: logits buffer required");
  const int BNsel = n_pad <= 32 ? 32 : (n_pad <= 64 ? 64 : (n_pad <= 128 ? 128 : 256));
  const long long T = static_cast<long long>(d.P) * d.S;
  CUtensorMap ta = make_tmap_bf16(x, dm, T, dm, kBM);
  CUtensorMap tb = make_tmap_bf16(wg, dm, static_cast<uint64_t>(d.P) * n_pad, dm, BNsel);
  GemmParams p{1, nullptr, nullptr, 0, n_pad, dm, 1, d.S, n_pad, d.P, 0, 1, 0, 0};
  GateEpiParams ep{o.logits, d.N, d.S};
  switch (BNsel) {
    case 32: launch_gemm<kModeGate, 32, false, false, EpiLogits>(ta, tb, p, ep, 0, s); break;
    case 64: launch_gemm<kModeGate, 64, false, false, EpiLogits>(ta, tb, p, ep, 0, s); break;
    case 128: launch_gemm<kModeGate, 128, false, false, EpiLogits>(ta, tb, p, ep, 0, s); break;
    default: launch_gemm<kModeGate, 256, false, false, EpiLogits>(ta, tb, p, ep, 0, s); break;
  }
  route_from_logits(o.logits, d, o, s);
}

}  // namespace tamoe
