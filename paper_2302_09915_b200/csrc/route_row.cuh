// Per-token routing shared by the fused gate epilogue and the standalone
// router: streaming top-k over fp64 probabilities with the reference's order
// (probability desc, expert index asc: gate.cpp:117-122), gate values
// (gate.cpp:124-134), per-warp expert histograms and probability sums
// (gate.cpp:115, reduced later in fixed order).
#pragma once
#include <cstdint>

#include "route.hpp"

namespace tamoe {

template <int KM = kMaxTopK>
struct TopK {
  double p[KM];
  int e[KM];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      p[j] = -1.0;
      e[j] = -1;
    }
  }
  // experts arrive in ascending index order, so a strict '>' keeps the lower index on ties
  __device__ __forceinline__ void insert(double cp, int ci, int k) {
    bool ins = false;
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      if (j < k) {
        const bool take = ins || (cp > p[j]);
        if (take) {
          const double tp = p[j];
          const int ti = e[j];
          p[j] = cp;
          e[j] = ci;
          cp = tp;
          ci = ti;
          ins = true;
        }
      }
    }
  }
};

// Reduce-scatter of 32 per-lane columns: on return lane c holds the warp-wide sum of column c
// (31 fp64 shuffles instead of 32 x 5).
__device__ __forceinline__ double warp_transpose_sum32(double (&v)[32], int lane) {
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool upper = (lane & h) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = upper ? v[i] : v[i + h];
      const double keep = upper ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return v[0];
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Finish one row: write picks and the warp's histogram row.  `valid` rows beyond S skip writes but
// still take part in the warp-wide ballots.
template <int KM>
__device__ __forceinline__ void finish_row(const TopK<KM>& tk, bool valid, long long gtok, int k, int N, int tile_warp,
                                           const RowRouteOut& o, int lane) {
  if (valid) {
    double mass = 0.0;
#pragma unroll
    for (int j = 0; j < KM; ++j)
      if (j < k) mass += tk.p[j];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      if (j < k) {
        const long long a = gtok * k + j;
        o.idx[a] = tk.e[j];
        o.score[a] = tk.p[j];
        const double g = k == 1 ? tk.p[j] : tk.p[j] / mass;
        o.gate[a] = static_cast<float>(g);
        if (o.gate64) o.gate64[a] = g;
      }
    }
  }
  int* h = o.hist4 + static_cast<long long>(tile_warp) * N;
  for (int e = 0; e < N; ++e) {
    bool hit = false;
#pragma unroll
    for (int j = 0; j < KM; ++j) hit |= (j < k) && (tk.e[j] == e);
    const unsigned bal = __ballot_sync(0xffffffffu, valid && hit);
    if (lane == 0) h[e] = __popc(bal);
  }
}

}  // namespace tamoe
