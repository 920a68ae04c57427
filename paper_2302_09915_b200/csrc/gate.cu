// Fused gate: logits = x . Wg^T on tcgen05 (TMA-staged, fp32 accumulate in
// TMEM), then per token in the epilogue: fp64 softmax exactly as the reference
// (max-subtract, exp, sequential sum over experts, divide: gate.cpp:12-28),
// streaming top-k (gate.cpp:117-134), per-warp expert histograms and
// probability partial sums for the aux loss (gate.cpp:115).
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
  RowRouteOut o;
  int N, k, S, TB;
};

// The two epilogue warps of a TMEM lane quarter (h = 0, 1) split each token row's experts: warp h owns
// 32-column chunks [h*C0, min(C, (h+1)*C0)).  Row max, the softmax denominator (sum of the two halves'
// sequential partial sums) and the top-k lists are exchanged through shared memory under a named barrier
// per lane quarter; warp h = 0 merges the lists (its experts have the lower indices, so ties keep it).
template <int KM>
struct EpiGate {
  using Params = GateEpiParams;
  struct Xchg {
    float mx[2][32];
    int fin[2][32];
    double sum[2][32];
    double tp[32][KM];
    int te[32][KM];
  };
  static constexpr int kWarpBytes = ((static_cast<int>(sizeof(Xchg)) + 127) / 128) * 128;
  static __device__ __forceinline__ void finish(const Params&, int) {}
  static __device__ __forceinline__ void prefetch(const Params&, const GemmParams&, const TileInfo&, int, int, int,
                                                  uint8_t*, const int*) {}
  static __device__ __forceinline__ void run(const Params& e, const GemmParams& p, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int h, int lane, uint8_t* wsm, const int*) {
    // the lane quarter's exchange area lives in warp q's (h = 0) scratch
    Xchg& X = *reinterpret_cast<Xchg*>(h == 0 ? wsm : wsm - 4 * kWarpBytes);
    const uint32_t bar_id = 1 + q;
    const int row = q * 32 + lane;
    const int tok = ti.m0 + row;
    const bool valid = tok < e.S;
    const long long gtok = static_cast<long long>(ti.g) * e.S + tok;
    const int tile_warp = (ti.g * e.TB + ti.m0 / kBM) * 4 + q;
    const int N = e.N;
    const int C = (N + 31) / 32, C0 = (C + 1) / 2;
    const int cb = h == 0 ? 0 : C0, ce = h == 0 ? C0 : C;
    // pass 1: max over my columns (and the non-finite check of gate.cpp:16); logits out
    float mx = -INFINITY;
    bool finite = true;
    for (int ch = cb; ch < ce; ++ch) {
      const int c0 = ch * 32;
      float v[32];
      load_acc32(tmem_tile, c0, v);
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        if (c0 + c < N) {
          finite &= isfinite(v[c]);
          mx = fmaxf(mx, v[c]);
        }
      }
      if (valid && e.o.logits) {
        float* dst = e.o.logits + gtok * N + c0;
        if (c0 + 32 <= N && (N % 4) == 0) {
#pragma unroll
          for (int c = 0; c < 32; c += 4) *reinterpret_cast<float4*>(dst + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (c0 + c < N) dst[c] = v[c];
        }
      }
    }
    X.mx[h][lane] = mx;
    X.fin[h][lane] = finite ? 1 : 0;
    ptx::named_bar_sync(bar_id, 64);
    mx = fmaxf(X.mx[0][lane], X.mx[1][lane]);
    finite = X.fin[0][lane] && X.fin[1][lane];
    if (h == 0 && valid && !finite) atomicOr(e.o.bad, 1);
    const double dmx = valid ? static_cast<double>(mx) : 0.0;
    // pass 2: my half of the denominator, sequential in expert order
    double part = 0.0;
    for (int ch = cb; ch < ce; ++ch) {
      const int c0 = ch * 32;
      float v[32];
      load_acc32(tmem_tile, c0, v);
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c0 + c < N) part += valid ? exp(static_cast<double>(v[c]) - dmx) : 0.0;
    }
    X.sum[h][lane] = part;
    ptx::named_bar_sync(bar_id, 64);
    const double denom = X.sum[0][lane] + X.sum[1][lane];
    // pass 3: probabilities, my top-k, probability sums of my columns
    TopK<KM> tk;
    tk.init();
    double* msum = e.o.msum4 + static_cast<long long>(tile_warp) * N;
    for (int ch = cb; ch < ce; ++ch) {
      const int c0 = ch * 32;
      float v[32];
      double pr[32];
      load_acc32(tmem_tile, c0, v);
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        pr[c] = (valid && c0 + c < N) ? exp(static_cast<double>(v[c]) - dmx) / denom : 0.0;
        if (c0 + c < N) {
          if (valid && e.o.probs) e.o.probs[gtok * N + c0 + c] = pr[c];
          tk.insert(pr[c], c0 + c, e.k);
        }
      }
      const double colsum = warp_transpose_sum32(pr, lane);
      if (c0 + lane < N) msum[c0 + lane] = colsum;
    }
    if (h == 1) {
#pragma unroll
      for (int j = 0; j < KM; ++j) {
        X.tp[lane][j] = tk.p[j];
        X.te[lane][j] = tk.e[j];
      }
    }
    ptx::named_bar_sync(bar_id, 64);
    if (h == 0) {
#pragma unroll
      for (int j = 0; j < KM; ++j)
        if (X.te[lane][j] >= 0) tk.insert(X.tp[lane][j], X.te[lane][j], e.k);
      finish_row(tk, valid, gtok, e.k, N, tile_warp, e.o, lane);
    }
    ptx::named_bar_sync(bar_id, 64);  // exchange area free for the next tile
  }
};

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

template <int BN>
static void gate_launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                        const GateEpiParams& ep, cudaStream_t s) {
  if (ep.k == 1) {
    launch_gemm<kModeGate, BN, false, false, EpiGate<1>>(ta, tb, p, ep, 0, s);
  } else if (ep.k == 2) {
    launch_gemm<kModeGate, BN, false, false, EpiGate<2>>(ta, tb, p, ep, 0, s);
  } else {
    launch_gemm<kModeGate, BN, false, false, EpiGate<kMaxTopK>>(ta, tb, p, ep, 0, s);
  }
}

void gate_forward(const __nv_bfloat16* x, const __nv_bfloat16* wg, int n_pad, const RouteDims& d, int dm,
                  const RowRouteOut& o, cudaStream_t s) {
  require(d.k >= 1 && d.k <= kMaxTopK && d.k <= d.N, "k must be in [1, min(N, 8)]");
  require(dm % 64 == 0, "gate: d must be a multiple of 64 (pad with zeros)");
  require(n_pad % 16 == 0 && n_pad >= d.N && n_pad <= 256, "gate: n_pad must be round_up(N, 16) <= 256");
  const int BNsel = n_pad <= 32 ? 32 : (n_pad <= 64 ? 64 : (n_pad <= 128 ? 128 : 256));
  const long long T = static_cast<long long>(d.P) * d.S;
  CUtensorMap ta = make_tmap_bf16(x, dm, T, dm, kBM);
  CUtensorMap tb = make_tmap_bf16(wg, dm, static_cast<uint64_t>(d.P) * n_pad, dm, BNsel);
  GemmParams p{1, nullptr, nullptr, 0, n_pad, dm, 1, d.S, n_pad, d.P, 0, 1, 0, 0};
  GateEpiParams ep{o, d.N, d.k, d.S, d.TB};
  switch (BNsel) {
    case 32: gate_launch<32>(ta, tb, p, ep, s); break;
    case 64: gate_launch<64>(ta, tb, p, ep, s); break;
    case 128: gate_launch<128>(ta, tb, p, ep, s); break;
    default: gate_launch<256>(ta, tb, p, ep, s); break;
  }
}

}  // namespace tamoe
