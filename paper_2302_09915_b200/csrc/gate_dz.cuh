// Per-token gate backward (trainer.cpp:318-345, gate.cpp:257-287), shared by the standalone gate dz kernel and
// the combine kernel it is fused into: softmax of the stored fp32 logits, the combine-weight Jacobian of dL/dg
// (top-1: dpi[e0] += dldg; top-k: renormalisation Jacobian with the raw scores), + (w / P) * coeff (topology or
// balance coefficients of the kept counts, stop-gradient), dz = p * (dpi - <dpi, p>).  One warp per token,
// expert e on lane e % 32.
#pragma once
#include <cuda_bf16.h>

#include "gate_bwd.hpp"
#include "route.hpp"

namespace tamoe {

// coeff[P*N] (shared memory, every thread of the block calls; the caller synchronises)
__device__ __forceinline__ void dz_coeff_smem(const GateDzArgs& a, double* coeff) {
  const int N = a.N;
  const double s2 = static_cast<double>(a.S) * a.S;
  for (int i = threadIdx.x; i < a.P * N; i += blockDim.x) {
    const double c = static_cast<double>(a.counts[i]);
    coeff[i] = a.aux_kind == 1 ? (static_cast<double>(N) * a.P_global / s2) * a.penalties[i] * c : c / s2;
  }
}

// loss finalisation (one warp): task = sum residual^2 / (P S d_out); aux = mean over processes.  The task
// partials (one per combine block: 4,096 at C2) are summed eight independent loads at a time per lane, in a
// fixed order (deterministic), so the warp is not a chain of dependent L2 round trips.
__device__ __forceinline__ void dz_finalize_losses(const GateDzArgs& a, int lane) {
  const int N = a.N;
  double task = 0.0;
  {
    constexpr int kU = 8;
    int i = lane;
    for (; i + 32 * (kU - 1) < a.n_loss_part; i += 32 * kU) {
      double v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = a.loss_part[i + 32 * u];
#pragma unroll
      for (int u = 0; u < kU; ++u) task += v[u];
    }
    for (; i < a.n_loss_part; i += 32) task += a.loss_part[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) task += __shfl_xor_sync(0xffffffffu, task, o);
  double aux = 0.0;
  for (int pr = 0; pr < a.P; ++pr) {
    double l = 0.0;
    for (int e = lane; e < N; e += 32) {
      const double frac = static_cast<double>(a.counts[pr * N + e]) / a.S;
      l += (a.aux_kind == 1 ? a.penalties[pr * N + e] : 1.0) * a.mean_probs[pr * N + e] * frac;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    aux += a.aux_kind == 1 ? static_cast<double>(N) * a.P_global * l : l;
  }
  if (lane == 0) {
    a.losses[0] = task / (static_cast<double>(a.P_global) * a.S * a.dout);
    a.losses[1] = aux / a.P_global;
  }
}

// The same finalisation by a whole block (blockDim a multiple of 32, <= 1024): the task partials are split over
// all threads (strided, eight loads in flight), reduced per warp and then across warps in a fixed order.
__device__ __forceinline__ void dz_finalize_losses_block(const GateDzArgs& a) {
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double task = 0.0;
  {
    constexpr int kU = 8;
    const int nt = blockDim.x;
    int i = threadIdx.x;
    for (; i + nt * (kU - 1) < a.n_loss_part; i += nt * kU) {
      double v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = a.loss_part[i + nt * u];
#pragma unroll
      for (int u = 0; u < kU; ++u) task += v[u];
    }
    for (; i < a.n_loss_part; i += nt) task += a.loss_part[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) task += __shfl_xor_sync(0xffffffffu, task, o);
  if (lane == 0) red[w] = task;
  __syncthreads();
  if (w == 0) {
    double t = 0.0;
    for (int i = 0; i < nw; ++i) t += red[i];
    const int N = a.N;
    double aux = 0.0;
    for (int pr = 0; pr < a.P; ++pr) {
      double l = 0.0;
      for (int e = lane; e < N; e += 32) {
        const double frac = static_cast<double>(a.counts[pr * N + e]) / a.S;
        l += (a.aux_kind == 1 ? a.penalties[pr * N + e] : 1.0) * a.mean_probs[pr * N + e] * frac;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
      aux += a.aux_kind == 1 ? static_cast<double>(N) * a.P_global * l : l;
    }
    if (lane == 0) {
      a.losses[0] = t / (static_cast<double>(a.P_global) * a.S * a.dout);
      a.losses[1] = aux / a.P_global;
    }
  }
}

template <int NPL>
__device__ __forceinline__ void dz_load_logits(const GateDzArgs& a, long long t, int lane, float (&l)[NPL]) {
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int e = lane + 32 * i;
    l[i] = e < a.N ? a.logits[t * a.N + e] : -INFINITY;
  }
}

// l: this lane's logits of token t (dz_load_logits, issued early so the load latency overlaps other work)
template <int KM, int NPL>
__device__ __forceinline__ void dz_token(const GateDzArgs& a, const double* coeff, long long t, int k, int lane,
                                         const float (&l)[NPL], const int (&ex_in)[KM], const float (&dl_in)[KM],
                                         const double (&sc_in)[KM]) {
  const int N = a.N;
  const int proc = static_cast<int>(t / a.S);
  // softmax of the stored fp32 logits (fp32 math, max-subtracted)
  float p[NPL], dpi[NPL];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < NPL; ++i) mx = fmaxf(mx, l[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float den = 0.f;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    p[i] = (lane + 32 * i < N) ? expf(l[i] - mx) : 0.f;
    den += p[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
  const float inv = 1.f / den;
  const float aux_scale = static_cast<float>(a.aux_weight / a.P_global);
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int e = lane + 32 * i;
    p[i] *= inv;
    dpi[i] = e < N ? aux_scale * static_cast<float>(coeff[proc * N + e]) : 0.f;
  }
  // combine-weight Jacobian (trainer.cpp:318-331)
  int ex[KM];
  float add[KM];
  if (k == 1) {
    ex[0] = ex_in[0];
    add[0] = dl_in[0];
#pragma unroll
    for (int j = 1; j < KM; ++j) {
      ex[j] = -1;
      add[j] = 0.f;
    }
  } else {
    double sc[KM], dg[KM];
    double mass = 0.0;
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      ex[j] = ex_in[j];
      sc[j] = sc_in[j];
      dg[j] = static_cast<double>(dl_in[j]);
      mass += sc[j];
    }
    const double inv2 = 1.0 / (mass * mass);
#pragma unroll
    for (int l2 = 0; l2 < KM; ++l2) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < KM; ++j)
        if (dg[j] != 0.0) acc += dg[j] * ((j == l2 ? mass : 0.0) - sc[j]) * inv2;
      add[l2] = static_cast<float>(acc);
    }
  }
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int e = lane + 32 * i;
#pragma unroll
    for (int j = 0; j < KM; ++j) dpi[i] += (ex[j] == e) ? add[j] : 0.f;
  }
  float dot = 0.f;
#pragma unroll
  for (int i = 0; i < NPL; ++i) dot += dpi[i] * p[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  __nv_bfloat16* dz = a.dz + t * a.n64;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int e = lane + 32 * i;
    if (e < a.n64) dz[e] = __float2bfloat16(e < N ? p[i] * (dpi[i] - dot) : 0.f);
  }
  // experts beyond 32 * NPL (n64 padding) are zero
  for (int e = 32 * NPL + lane; e < a.n64; e += 32) dz[e] = __float2bfloat16(0.f);
}

}  // namespace tamoe
