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
#include <cstdlib>

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

// Fused gate (N <= 64 experts): the GEMM epilogue routes its 128 tokens in place -- the logits never
// round-trip through a separate kernel.  Lane = token; the two epilogue warps of a TMEM lane quarter split the
// experts (column half h holds experts 32h..32h+31 of its 32 tokens, N <= 32: half 0 alone).  Per token,
// exactly as the reference (gate.cpp:12-28): max, fp64 exp(v - max), the denominator summed sequentially in
// expert order (half 0's partial sum handed to half 1 through shared memory), p = e / denominator correctly
// rounded.  Top-k in (p desc, expert asc) order (gate.cpp:117-122): division is monotone, so the top-k by e
// are found first (per half, then merged) and only the candidates within a few ulps of the k-th are divided
// exactly -- the selected p (score, gate value) are the reference's bits.  Column sums of the 32-token group
// (mean probabilities, gate.cpp:115) use e * (1 / denominator) reduced across lanes in a fixed butterfly
// order; expert histograms by ballot.  fp32 logits are still stored (the backward recomputes the softmax).
struct GateRouteParams {
  float* logits;
  RowRouteOut o;
  int N, S, k, TB;
  int probe;  // A/B probe (TAMOE_GATE_PROBE): 1 = release TMEM and stop, 2 = skip the fp64 exp
};

template <int KM>
struct RouteXchg {  // per-warp, per-lane exchange record between the two halves of a lane quarter
  float mx[32];
  int fin[32];
  double sum[32];       // half 0: partial denominator (experts 0-31); half 1: the full denominator
  double te_p[KM][32];  // this half's top-k by e, then (after the candidates pass) by exact p
  int te_e[KM][32];
};

template <int KM>
__device__ __forceinline__ void merge_topk(const double* pa, const int* ea, const double* pb, const int* eb, int k,
                                           TopK<KM>& out) {
  // two lists sorted by (value desc, expert asc); every expert of list a is below every expert of list b, so on
  // equal values a wins
  int ia = 0, ib = 0;
#pragma unroll
  for (int j = 0; j < KM; ++j) {
    if (j < k) {
      const double va = ia < k ? pa[ia] : -2.0, vb = ib < k ? pb[ib] : -2.0;
      if (va >= vb) {
        out.p[j] = va;
        out.e[j] = ea[ia];
        ++ia;
      } else {
        out.p[j] = vb;
        out.e[j] = eb[ib];
        ++ib;
      }
    }
  }
}

// Branch-free fp64 exp for x <= 0 (the softmax's exp(v - max)): x clamped to >= -700 (exp(-700) ~ 1e-304 vanishes
// against the denominator >= 1 either way), n = round(x / ln2) by the 1.5 * 2^52 shift, r = x - n ln2 with a
// 32-bit-exact high part of ln2 (|r| <= ln2 / 2), Taylor to degree 13 (truncation < 5e-18 relative), and 2^n
// applied to the exponent field.  Within 1 ulp of the correctly rounded value, like CUDA's exp(), but with no
// special-case branch, so the 32 exponentials of a lane interleave.
template <int W>
__device__ __forceinline__ void exp_nonpos_x(double (&x)[W]) {
  // W independent evaluations written in lockstep, so the dependent DFMA chains interleave
  const double shift = 6755399441055744.0;  // 1.5 * 2^52
  double n[W], r[W], p[W];
  int ni[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const double xc = fmax(x[w], -700.0);
    const double t = fma(xc, 0x1.71547652b82fep+0, shift);
    n[w] = t - shift;
    ni[w] = __double2loint(t);
    r[w] = fma(n[w], -0x1.62e42fee00000p-1, xc);
  }
#pragma unroll
  for (int w = 0; w < W; ++w) r[w] = fma(n[w], -0x1.a39ef35793c76p-33, r[w]);
  constexpr double c[13] = {0x1.1eed8eff8d898p-29, 0x1.ae64567f544e4p-26, 0x1.27e4fb7789f5cp-22,
                            0x1.71de3a556c734p-19, 0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-13,
                            0x1.6c16c16c16c17p-10, 0x1.1111111111111p-7,  0x1.5555555555555p-5,
                            0x1.5555555555555p-3,  0.5,                   1.0,
                            1.0};
#pragma unroll
  for (int w = 0; w < W; ++w) p[w] = fma(0x1.6124613a86d09p-33, r[w], c[0]);
#pragma unroll
  for (int j = 1; j < 13; ++j)
#pragma unroll
    for (int w = 0; w < W; ++w) p[w] = fma(p[w], r[w], c[j]);
#pragma unroll
  for (int w = 0; w < W; ++w) x[w] = __hiloint2double(__double2hiint(p[w]) + (ni[w] << 20), __double2loint(p[w]));
}

template <int NC, int KM>
struct EpiRoute {
  using Params = GateRouteParams;
  static constexpr bool kEarlyRelease = true;
  static constexpr int kWarpBytes = (sizeof(RouteXchg<KM>) + 127) / 128 * 128;
  static __device__ __forceinline__ void finish(const Params&, int) {}
  static __device__ __forceinline__ void prefetch(const Params&, const GemmParams&, const TileInfo&, int, int, int,
                                                  uint8_t*, const int*) {}
  template <class Release>
  static __device__ __forceinline__ void run(const Params& e, const GemmParams&, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int h, int lane, uint8_t* wsm, const int*,
                                             Release&& release) {
    constexpr bool kTwo = NC == 64;  // two halves cooperate
    if (!kTwo && h != 0) {
      release();
      return;
    }
    RouteXchg<KM>& me = *reinterpret_cast<RouteXchg<KM>*>(wsm);
    RouteXchg<KM>& pa = *reinterpret_cast<RouteXchg<KM>*>(h == 0 ? wsm + 4 * kWarpBytes : wsm - 4 * kWarpBytes);
    auto pair_sync = [&]() {
      if constexpr (kTwo) ptx::named_bar_sync(1 + q, 64);
    };
    const int N = e.N, k = e.k;
    const int cb = 32 * h;  // first expert of this half
    const int tok = ti.m0 + q * 32 + lane;
    const bool valid = tok < e.S;
    const long long gtok = static_cast<long long>(ti.g) * e.S + tok;
    float v[32];
    {
      uint32_t r[32];
      ptx::tmem_ld_32x32b_x32(tmem_tile + cb, r);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
    }
    release();
    if (e.probe == 1) return;
    if (valid) {
      float* dst = e.logits + gtok * N + cb;
      if ((N & 3) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          if (cb + i < N) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (cb + i < N) dst[i] = v[i];
      }
    }
    float mx = -INFINITY;
    bool finite = true;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (cb + i < N) {
        finite &= isfinite(v[i]);
        mx = fmaxf(mx, v[i]);
      }
    if constexpr (kTwo) {  // barrier 1: row max and finiteness of both halves
      me.mx[lane] = mx;
      me.fin[lane] = finite;
      pair_sync();
      mx = fmaxf(mx, pa.mx[lane]);
      finite = finite && pa.fin[lane];
    }
    const bool ok = finite || !valid;
    const double dmx = static_cast<double>(mx);
    double E[32];
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += 4) {
      double xs[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) xs[w] = static_cast<double>(cb + i0 + w < N ? v[i0 + w] : mx) - dmx;
      exp_nonpos_x<4>(xs);
#pragma unroll
      for (int w = 0; w < 4; ++w) E[i0 + w] = (cb + i0 + w < N && ok) ? xs[w] : 0.0;
    }
    if (e.probe == 3) {  // stop after the exps
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += E[i];
      if (valid) e.o.msum4[gtok] = acc;
      return;
    }
    // top-k by e of this half (experts ascending: strict '>' keeps the lower one on ties)
    TopK<KM> te;
    te.init();
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (cb + i < N) te.insert(E[i], cb + i, k);
    // denominator in expert order: half 0 sums experts 0-31, half 1 continues from that partial sum
    double den = 0.0;
    if (h == 0) {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < N) den += E[i];
    }
    // merged top-k by e (both halves hold it after barrier 2)
    TopK<KM> m;
    if constexpr (kTwo) {  // barrier 2: half 0's partial sum and both halves' top-k by e
      if (h == 0) me.sum[lane] = den;
#pragma unroll
      for (int j = 0; j < KM; ++j) {
        me.te_p[j][lane] = te.p[j];
        me.te_e[j][lane] = te.e[j];
      }
      pair_sync();
      if (h == 1) {
        den = pa.sum[lane];
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (32 + i < N) den += E[i];
      }
      double ap[KM], bp[KM];
      int ae[KM], be[KM];
      const RouteXchg<KM>& h0 = h == 0 ? me : pa;
      const RouteXchg<KM>& h1 = h == 0 ? pa : me;
#pragma unroll
      for (int j = 0; j < KM; ++j) {
        ap[j] = h0.te_p[j][lane];
        ae[j] = h0.te_e[j][lane];
        bp[j] = h1.te_p[j][lane];
        be[j] = h1.te_e[j][lane];
      }
      merge_topk<KM>(ap, ae, bp, be, k, m);
    } else {
      m = te;
    }
    double kth = m.p[0];
#pragma unroll
    for (int j = 0; j < KM; ++j)
      if (j < k) kth = m.p[j];
    // Division is monotone, so the top-k by p is the top-k by e unless an expert with a smaller e rounds to the
    // same p as a selected one and has the lower index (the reference breaks p ties by index).  Only experts with
    // e within a few ulps of the k-th can: flag them (no division on the common path).
    const double thr = kth * (1.0 - 0x1p-46);
    bool extra = false;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      bool sel = false;
#pragma unroll
      for (int j = 0; j < KM; ++j) sel |= (j < k) && (m.e[j] == cb + i);
      extra |= (cb + i < N) && !sel && E[i] >= thr;
    }
    bool any_extra = __any_sync(0xffffffffu, extra);
    if constexpr (kTwo) {  // barrier 3: the full denominator (half 1) and the extra flags to both halves
      pair_sync();  // both halves are done reading the top-k lists
      if (h == 1) me.sum[lane] = den;
      me.fin[lane] = any_extra;
      pair_sync();
      if (h == 0) den = pa.sum[lane];
      any_extra = any_extra || pa.fin[lane];
    }
    TopK<KM> tp;
    if (!any_extra) {
      // common path: exactly the k selected are divided (warp-uniform, no divergence)
      tp = m;
#pragma unroll
      for (int j = 0; j < KM; ++j)
        if (j < k) tp.p[j] = m.p[j] / den;
      // two selected e may round to the same p: restore (p desc, expert asc) among the selected
#pragma unroll
      for (int j = 1; j < KM; ++j)
#pragma unroll
        for (int i = j; i > 0; --i)
          if (i < k && (tp.p[i] > tp.p[i - 1] || (tp.p[i] == tp.p[i - 1] && tp.e[i] < tp.e[i - 1]))) {
            const double tpv = tp.p[i];
            tp.p[i] = tp.p[i - 1];
            tp.p[i - 1] = tpv;
            const int tev = tp.e[i];
            tp.e[i] = tp.e[i - 1];
            tp.e[i - 1] = tev;
          }
    } else {
      // near-tie path (pair-uniform): exact p for every candidate of this half in expert order, then merged
      tp.init();
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (cb + i < N && E[i] >= thr) tp.insert(E[i] / den, cb + i, k);
      if constexpr (kTwo) {  // barrier 4: half 1's candidates to half 0, which merges
        if (h == 1) {
#pragma unroll
          for (int j = 0; j < KM; ++j) {
            me.te_p[j][lane] = tp.p[j];
            me.te_e[j][lane] = tp.e[j];
          }
        }
        pair_sync();
        if (h == 0) {
          double bp[KM];
          int be[KM];
#pragma unroll
          for (int j = 0; j < KM; ++j) {
            bp[j] = pa.te_p[j][lane];
            be[j] = pa.te_e[j][lane];
          }
          TopK<KM> mm;
          merge_topk<KM>(tp.p, tp.e, bp, be, k, mm);
          tp = mm;
        }
      }
    }
    if (e.probe == 5) {  // stop after the exact candidates / merge
      if (valid) e.o.msum4[gtok] = tp.p[0] + tp.e[0];
      return;
    }
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    // 32-token group slot of this warp (= route_logits' block index)
    const long long slot = (static_cast<long long>(ti.g) * e.TB + ti.m0 / kRouteTile) * 4 + q;
    if (h == 0) {
      if (!ok) {  // non-finite logit: experts 0..k-1, NaN gates, poisoned column sums (see route_logits_kernel)
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          tp.p[j] = 0.0;
          tp.e[j] = j;
        }
      }
      if (valid) {
        double mass = 0.0;
#pragma unroll
        for (int j = 0; j < KM; ++j)
          if (j < k) mass += tp.p[j];
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          if (j < k) {
            const long long a = gtok * k + j;
            e.o.idx[a] = tp.e[j];
            e.o.score[a] = tp.p[j];
            const double g = !ok ? qnan : (k == 1 ? tp.p[j] : tp.p[j] / mass);
            e.o.gate[a] = static_cast<float>(g);
            if (e.o.gate64) e.o.gate64[a] = g;
          }
        }
      }
      if (__any_sync(0xffffffffu, !ok)) {
        if (lane == 0) {
          atomicOr(e.o.bad, 1);
          if (e.o.bad_host) *reinterpret_cast<volatile int*>(e.o.bad_host) = 1;
        }
      }
      // expert histogram of the group's picks (all N columns): lane c % 32 keeps column c's count
      int cnt0 = 0, cnt1 = 0;
#pragma unroll 4
      for (int c = 0; c < N; ++c) {
        bool hit = false;
#pragma unroll
        for (int t = 0; t < KM; ++t) hit |= (t < k) && (tp.e[t] == c);
        const int n = __popc(__ballot_sync(0xffffffffu, valid && hit));
        if (lane == (c & 31)) {
          if (c < 32) cnt0 = n;
          else cnt1 = n;
        }
      }
      if (lane < N) e.o.hist4[slot * N + lane] = cnt0;
      if (32 + lane < N) e.o.hist4[slot * N + 32 + lane] = cnt1;
    }
    if (e.probe == 6) return;  // stop before the column sums
    // column sums of p = e * (1 / den) over the group's 32 tokens for this half's experts (fixed butterfly)
    const double rcp = valid ? (ok ? 1.0 / den : qnan) : 0.0;
#pragma unroll
    for (int i = 0; i < 32; ++i) E[i] *= rcp;
    const double sum = warp_transpose_sum32(E, lane);
    if (cb + lane < N) e.o.msum4[slot * N + cb + lane] = sum;
    pair_sync();  // exchange slots free for the next tile
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
  ptx::pdl_trigger();
  ptx::pdl_wait();
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
    if (any_bad) {
      atomicOr(o.bad, 1);
      if (o.bad_host) *reinterpret_cast<volatile int*>(o.bad_host) = 1;
    }
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
  launch_pdl(route_logits_kernel<EPL, KM>, static_cast<unsigned>(d.tiles()) * 4, kRouteGroupWarps * 32, smem, s,
             logits, d, o);
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

// TAMOE_FUSED_GATE=0: logits GEMM + the separate router kernel (A/B switch)
static bool fused_gate_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("TAMOE_FUSED_GATE");
    return !(v && v[0] == '0');
  }();
  return on;
}

bool gate_is_fused(int N, bool want_probs) { return fused_gate_enabled() && N <= 64 && !want_probs; }

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
  GemmParams p{1, nullptr, nullptr, 0, n_pad, dm, 1, d.S, n_pad, d.P, 0, 1};
  if (gate_is_fused(d.N, o.probs != nullptr)) {
    // one launch: logits GEMM + per-token routing in the epilogue
    static const int probe = [] {
      const char* v = std::getenv("TAMOE_GATE_PROBE");
      return v ? std::atoi(v) : 0;
    }();
    GateRouteParams rp{o.logits, o, d.N, d.S, d.k, d.TB, probe};
    const int km = d.k == 1 ? 1 : (d.k == 2 ? 2 : kMaxTopK);
#define TAMOE_GATE_ROUTE(NC, KM) launch_gemm<kModeGate, NC, false, false, EpiRoute<NC, KM>>(ta, tb, p, rp, 0, s)
    if (BNsel == 32) {
      if (km == 1) TAMOE_GATE_ROUTE(32, 1);
      else if (km == 2) TAMOE_GATE_ROUTE(32, 2);
      else TAMOE_GATE_ROUTE(32, kMaxTopK);
    } else {
      if (km == 1) TAMOE_GATE_ROUTE(64, 1);
      else if (km == 2) TAMOE_GATE_ROUTE(64, 2);
      else TAMOE_GATE_ROUTE(64, kMaxTopK);
    }
#undef TAMOE_GATE_ROUTE
    return;
  }
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
