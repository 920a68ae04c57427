// Gate backward (trainer.cpp:318-355, gate.cpp:257-287):
//   dpi_t  = combine-weight Jacobian of dldg (top-1: dpi[e0] += dldg; top-k: renormalisation
//            Jacobian with the raw scores) + (w / P) * coeff  (coeff = topo or balance coefficients
//            of the kept counts, stop-gradient);
//   dz_t   = pi_t * (dpi_t - <dpi_t, pi_t>)                          (softmax backward)
//   dWg    = x^T dz            (tcgen05, split-K over tokens, fixed-order reduction)
//   dX     = dz Wg + sum_slots dX_perm[pos]     (tcgen05 GEMM whose epilogue gathers the expert
//                                                path's input gradient back to token order)
// plus the loss finalisation (task MSE, aux loss: trainer.cpp:334-345, 360-361).
#include <cstdlib>
#include <cuda_bf16.h>

#include <cmath>

#include "common.hpp"
#include "gate_bwd.hpp"
#include "gate_dz.cuh"
#include "gemm_launch.cuh"
#include "route.hpp"
#include "tma_host.hpp"

namespace tamoe {

namespace {

constexpr int kDzWarps = 8;
constexpr int kMaxNPerLane = 8;  // N <= 256

// KT: compile-time top-k (0 = runtime k <= 8); NPL: experts per lane (N <= 32 * NPL).
template <int KT, int NPL>
__global__ void __launch_bounds__(kDzWarps * 32) gate_dz_kernel(const __grid_constant__ GateDzArgs a) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  constexpr int KM = KT > 0 ? KT : kMaxTopK;
  extern __shared__ double coeff[];  // [P*N]
  dz_coeff_smem(a, coeff);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < 32) dz_finalize_losses(a, threadIdx.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t = static_cast<long long>(blockIdx.x) * kDzWarps + warp;
  if (t >= static_cast<long long>(a.P) * a.S) return;
  const int k = KT > 0 ? KT : a.k;
  // every per-token load up front (independent of the softmax below), so their latencies overlap
  int ex_in[KM];
  float dl_in[KM];
  double sc_in[KM];
#pragma unroll
  for (int j = 0; j < KM; ++j) {
    ex_in[j] = j < k ? a.idx[t * k + j] : -1;
    dl_in[j] = j < k ? a.dldg[t * k + j] : 0.f;
    sc_in[j] = (k > 1 && j < k) ? a.score[t * k + j] : 0.0;
  }
  float lg[NPL];
  dz_load_logits<NPL>(a, t, lane, lg);
  dz_token<KM, NPL>(a, coeff, t, k, lane, lg, ex_in, dl_in, sc_in);
}

template <int KT>
void launch_dz(const GateDzArgs& a, int blocks, cudaStream_t s) {
  const size_t smem = sizeof(double) * a.P * a.N;
  if (a.N <= 32) launch_pdl(gate_dz_kernel<KT, 1>, blocks, kDzWarps * 32, smem, s, a);
  else if (a.N <= 64) launch_pdl(gate_dz_kernel<KT, 2>, blocks, kDzWarps * 32, smem, s, a);
  else if (a.N <= 128) launch_pdl(gate_dz_kernel<KT, 4>, blocks, kDzWarps * 32, smem, s, a);
  else launch_pdl(gate_dz_kernel<KT, 8>, blocks, kDzWarps * 32, smem, s, a);
}

// dWg partials: acc[m = d index][n = expert] -> part[((ks * P + proc) * n64 + n) * d + m]
struct EpiGateDw {
  struct Params {
    float* part;
    int d, n64, P;
    int finalize;    // the loss finalisation of the gate dz pass fused into combine: one epilogue warp of CTA 0
    GateDzArgs fin;  // runs it before its first accumulator is ready (hidden under the mainloop)
  };
  static __device__ __forceinline__ void finish(const Params&, int) {}
  static __device__ __forceinline__ void prefetch(const Params& e, const GemmParams&, const TileInfo& ti, int q, int h,
                                                  int lane, uint8_t*, const int*) {
    if (e.finalize && blockIdx.x == 0 && q == 0 && h == 0 && ti.g == 0 && ti.ks == 0 && ti.m0 == 0 && ti.n0 == 0)
      dz_finalize_losses(e.fin, lane);
  }
  static __device__ __forceinline__ void run(const Params& e, const GemmParams& p, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int h, int lane, uint8_t*, const int*) {
    const int m = ti.m0 + q * 32 + lane;
    for (int c0 = 32 * h; c0 < ti.n; c0 += 64) {
      float v[32];
      if (ti.k_len > 0) {
        load_acc32(tmem_tile, c0, v);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const int n = ti.n0 + c0 + c;
        e.part[((static_cast<long long>(ti.ks) * e.P + ti.g) * e.n64 + n) * e.d + m] = v[c];
      }
    }
  }
};

__global__ void dwg_reduce_kernel(const float* __restrict__ part, int splits, int P, int n64, int n_pad, int d,
                                  int N, float* __restrict__ dwg) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const long long total = static_cast<long long>(P) * n_pad * d;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i % d);
    const int n = static_cast<int>((i / d) % n_pad);
    const int proc = static_cast<int>(i / (static_cast<long long>(d) * n_pad));
    float s = 0.f;
    if (n < N) {
      // eight partials in flight per thread, summed in split order (deterministic)
      const long long stride = static_cast<long long>(P) * n64 * d;
      const float* src = part + (static_cast<long long>(proc) * n64 + n) * d + m;
      int ks = 0;
      for (; ks + 8 <= splits; ks += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (ks + u) * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
      }
      for (; ks < splits; ++ks) s += __ldg(src + ks * stride);
    }
    dwg[i] = s;
  }
}

// dX: acc[token][d col] + gathered expert-path input gradients
struct GateDxParams {
  __nv_bfloat16* dx;
  PeerBufs dxp;      // expert-path input gradients in every owner's receive layout
  const int* pos;
  const int* idx;
  RowMap map;
  int k, S, d;
};

// KT = compile-time top-k (0: runtime k).  Warp h of a lane quarter owns the contiguous column half
// [128h, 128h + 128) of the tile, so each lane gathers 256 contiguous bytes of every expert-path row it
// needs -- all of them into registers before the first accumulator load, so their latency overlaps.
template <int KT>
struct EpiGateDx {
  using Params = GateDxParams;
  static constexpr int KM = KT > 0 ? KT : kMaxTopK;
  static __device__ __forceinline__ void finish(const Params&, int) {}
  static __device__ __forceinline__ void prefetch(const Params&, const GemmParams&, const TileInfo&, int, int, int,
                                                  uint8_t*, const int*) {}
  static __device__ __forceinline__ void add8(float* v, const uint4& w) {
    const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(hh[i]);
      v[2 * i] += f.x;
      v[2 * i + 1] += f.y;
    }
  }
  static __device__ __forceinline__ void run(const Params& e, const GemmParams& p, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int h, int lane, uint8_t*, const int*) {
    const int tok = ti.m0 + q * 32 + lane;
    const bool valid = tok < e.S;  // tcgen05.ld is warp-collective: every lane runs the loops
    const long long gtok = static_cast<long long>(ti.g) * e.S + tok;
    const int k = KT > 0 ? KT : e.k;
    // the expert-path gradient of pick gtok*k+j sits at that row of dxp (pushed back by the expert dgrad
    // epilogue): addresses are known up front; dropped picks (pos < 0, stale rows) are zeroed after the load
    const __nv_bfloat16* srcs[KM];
    bool keep[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      const bool in = valid && j < k;
      srcs[j] = in ? e.dxp.p[0] + (gtok * k + j) * e.d : nullptr;
      keep[j] = in && e.pos[gtok * k + j] >= 0;
    }
    constexpr int kCh = 4;  // BN = 256: four 32-column chunks per warp (every other chunk)
    if constexpr (KT > 0) {
      uint4 g[KM][kCh][4];
#pragma unroll
      for (int j = 0; j < KM; ++j)
#pragma unroll
        for (int c = 0; c < kCh; ++c)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            g[j][c][u] = srcs[j] ? reinterpret_cast<const uint4*>(srcs[j] + ti.n0 + 128 * h + 32 * c)[u]
                                 : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < KM; ++j)
        if (!keep[j])
#pragma unroll
          for (int c = 0; c < kCh; ++c)
#pragma unroll
            for (int u = 0; u < 4; ++u) g[j][c][u] = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < kCh; ++c) {
        const int c0 = 128 * h + 32 * c;
        float v[32];
        load_acc32(tmem_tile, c0, v);
#pragma unroll
        for (int j = 0; j < KM; ++j)
#pragma unroll
          for (int u = 0; u < 4; ++u) add8(v + 8 * u, g[j][c][u]);
        if (!valid) continue;
        store32(e, gtok, ti.n0 + c0, v);
      }
    } else {
      for (int c0 = 128 * h; c0 < min(ti.n, 128 * h + 128); c0 += 32) {
        float v[32];
        load_acc32(tmem_tile, c0, v);
#pragma unroll
        for (int j = 0; j < KM; ++j)
          if (keep[j])
#pragma unroll
            for (int u = 0; u < 4; ++u) add8(v + 8 * u, reinterpret_cast<const uint4*>(srcs[j] + ti.n0 + c0)[u]);
        if (!valid) continue;
        store32(e, gtok, ti.n0 + c0, v);
      }
    }
  }
  static __device__ __forceinline__ void store32(const Params& e, long long gtok, int col, const float* v) {
    uint4* dst = reinterpret_cast<uint4*>(e.dx + gtok * e.d + col);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint4 w;
      __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
      for (int i = 0; i < 4; ++i) hh[i] = __floats2bfloat162_rn(v[8 * u + 2 * i], v[8 * u + 2 * i + 1]);
      dst[u] = w;
    }
  }
};

// Tile-ahead variant for top-1 / top-2 (BN = 128; warp h owns the 64 columns [64h, 64h + 64) of its 32
// tokens).  The expert-path rows and their pos flags of tile i+1 stream into the warp's second staging buffer
// with cp.async (coalesced: 8 lanes per 128-byte row segment, 128-byte swizzled in shared memory) while tile
// i is finished; the sum is written back into the staging tile in place and leaves as one 4 KiB TMA store.
struct GateDxAheadParams {
  CUtensorMap out;   // dx [T x d], box {64, 32}, 128B swizzle (the staging layout)
  const __nv_bfloat16* dxp;
  const int* pos;
  int S, d;
};

template <int KT>
struct EpiGateDxAhead {
  using Params = GateDxAheadParams;
  static constexpr int kSlotBytes = 32 * 128;               // 32 tokens x 64 columns bf16
  static constexpr int kBufBytes = KT * kSlotBytes + 1024;  // + pos flags, 1 KiB aligned for the swizzle
  static constexpr int kWarpBytes = 2 * kBufBytes;
  static __device__ __forceinline__ void prefetch(const Params& e, const GemmParams&, const TileInfo& ti, int q, int h,
                                                  int lane, uint8_t* buf, const int*) {
    if (lane == 0) ptx::bulk_wait_read<0>();  // the store issued from this buffer two tiles ago has read it
    __syncwarp();
    const int tok0 = ti.m0 + q * 32;
    const long long g0 = static_cast<long long>(ti.g) * e.S + tok0;
    const int col0 = ti.n0 + 64 * h;
#pragma unroll
    for (int i = 0; i < 8 * KT; ++i) {
      const int id = i * 32 + lane;
      const int j = id >> 8, rr = (id >> 3) & 31, c = id & 7;
      const bool ok = tok0 + rr < e.S;
      const __nv_bfloat16* src = e.dxp + ((ok ? g0 + rr : 0) * KT + j) * e.d + col0 + 8 * c;
      ptx::cp_async_16(buf + j * kSlotBytes + rr * 128 + ((c ^ (rr & 7)) * 16), src, ok);
    }
    const bool ok = tok0 + lane < e.S;
    ptx::cp_async_small<4 * KT>(buf + KT * kSlotBytes + lane * 4 * KT, e.pos + (ok ? g0 + lane : 0) * KT, ok);
    ptx::cp_async_commit();
  }
  static __device__ __forceinline__ void prefetch_none() { ptx::cp_async_commit(); }
  static __device__ __forceinline__ void finish(const Params&, int lane) {
    ptx::cp_async_wait<0>();
    if (lane == 0) ptx::bulk_wait<0>();
    __syncwarp();
  }
  static __device__ __forceinline__ void run(const Params& e, const GemmParams&, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int h, int lane, uint8_t* buf, const int*) {
    ptx::cp_async_wait<1>();  // this tile's group (the next tile's may still be in flight)
    __syncwarp();
    const int* posf = reinterpret_cast<const int*>(buf + KT * kSlotBytes) + lane * KT;
    bool keep[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) keep[j] = posf[j] >= 0;  // dropped picks: their dxp rows are stale
    uint8_t* row = buf + lane * 128;
    const int sw = lane & 7;
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      float v[32];
      load_acc32(tmem_tile, 64 * h + 32 * cc, v);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int off = ((cc * 4 + u) ^ sw) * 16;
#pragma unroll
        for (int j = 0; j < KT; ++j)
          if (keep[j]) EpiGateDx<KT>::add8(v + 8 * u, *reinterpret_cast<const uint4*>(row + j * kSlotBytes + off));
        uint4 w;
        __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
        for (int i = 0; i < 4; ++i) hh[i] = __floats2bfloat162_rn(v[8 * u + 2 * i], v[8 * u + 2 * i + 1]);
        *reinterpret_cast<uint4*>(row + off) = w;  // in place: slot 0 becomes the output staging tile
      }
    }
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_store_2d(&e.out, buf, ti.n0 + 64 * h, static_cast<int>(static_cast<long long>(ti.g) * e.S + ti.m0 + q * 32));
      ptx::bulk_commit();
    }
  }
};

}  // namespace

void gate_dz(const GateDzArgs& a, cudaStream_t s) {
  require(a.N <= 32 * kMaxNPerLane, "gate backward: N must be <= 256");
  require(a.k >= 1 && a.k <= kMaxTopK, "gate backward: k out of range");
  const long long T = static_cast<long long>(a.P) * a.S;
  const int blocks = static_cast<int>((T + kDzWarps - 1) / kDzWarps);
  if (a.k == 1) launch_dz<1>(a, blocks, s);
  else if (a.k == 2) launch_dz<2>(a, blocks, s);
  else launch_dz<0>(a, blocks, s);
  TAMOE_CUDA(cudaGetLastError());
}

int gate_dw_splits(int P, int S, int d, int n64) {
  const int tiles_per_split = P * (d / 128) * (n64 / 64);
  int splits = (num_sms() + tiles_per_split - 1) / tiles_per_split;
  const int max_split = (S + 63) / 64;
  if (splits > max_split) splits = max_split;
  return splits < 1 ? 1 : splits;
}

void gate_dw(const __nv_bfloat16* x, const __nv_bfloat16* dz, int P, int S, int d, int n64, int n_pad, int N,
             float* part, int splits, float* dwg, cudaStream_t s, const GateDzArgs* finalize) {
  require(d % 128 == 0, "gate dW: d must be a multiple of 128");
  require(n64 % 64 == 0, "gate dW: dz width must be a multiple of 64");
  require(P == 1 || S % 16 == 0, "gate dW: S must be a multiple of 16 when several processes share a device");
  const long long T = static_cast<long long>(P) * S;
  CUtensorMap ta = make_tmap_bf16(x, d, T, d, 64);     // A = x^T (MN-major)
  CUtensorMap tb = make_tmap_bf16(dz, n64, T, n64, 64);  // B = dz   (MN-major)
  GemmParams p{1, nullptr, nullptr, d, 64, 0, splits, S, 0, P, 0, 1};
  // one 64-column N block per launch keeps BN = 64 (n64 > 64 loops over column blocks)
  EpiGateDw::Params ep{part, d, n64, P, finalize ? 1 : 0, finalize ? *finalize : GateDzArgs{}};
  if (n64 == 64) {
    launch_gemm<kModeGateDw, 64, true, true, EpiGateDw>(ta, tb, p, ep, 0, s);
  } else {
    require(n64 == 256 || n64 == 128, "gate dW: unsupported expert padding");
    if (n64 == 128) {
      p.Nw = 128;
      launch_gemm<kModeGateDw, 128, true, true, EpiGateDw>(ta, tb, p, ep, 0, s);
    } else {
      p.Nw = n64;
      launch_gemm<kModeGateDw, 256, true, true, EpiGateDw>(ta, tb, p, ep, 0, s);
    }
  }
  const long long total = static_cast<long long>(P) * n_pad * d;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 4096));
  launch_pdl(dwg_reduce_kernel, blocks, 256, 0, s, part, splits, P, n64, n_pad, d, N, dwg);
  TAMOE_CUDA(cudaGetLastError());
}

void gate_dx(const __nv_bfloat16* dz, const __nv_bfloat16* wg, int P, int S, int d, int n64, int n_pad,
             const PeerBufs& dxp, const int* pos, const int* idx, const RowMap& map, int k, __nv_bfloat16* dx,
             cudaStream_t s) {
  require(d % 256 == 0, "gate dX: d must be a multiple of 256");
  const long long T = static_cast<long long>(P) * S;
  CUtensorMap ta = make_tmap_bf16(dz, n64, T, n64, 128);                         // A = dz (K-major)
  CUtensorMap tb = make_tmap_bf16(wg, d, static_cast<uint64_t>(P) * n_pad, d, 64);  // B = Wg (MN-major)
  GemmParams p{1, nullptr, nullptr, 0, d, n_pad, 1, S, n_pad, P, 0, 1};
  // tile-ahead TMA path: top-1 / top-2, local expert-path rows, and 32-token warp groups that never straddle
  // two processes (the TMA store writes whole 32-row boxes; rows past T are clipped)
  static const bool ahead_on = [] {
    const char* v = std::getenv("TAMOE_GATE_DX_AHEAD");
    return !(v && v[0] == '0');
  }();
  if (ahead_on && (k == 1 || k == 2) && map.P == 1 && (P == 1 || S % 32 == 0)) {
    GateDxAheadParams ea{make_tmap_bf16_box(dx, d, T, d, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B), dxp.p[0], pos, S, d};
    if (k == 1) launch_gemm<kModeGateDx, 128, false, true, EpiGateDxAhead<1>>(ta, tb, p, ea, 0, s);
    else launch_gemm<kModeGateDx, 128, false, true, EpiGateDxAhead<2>>(ta, tb, p, ea, 0, s);
    return;
  }
  GateDxParams ep{dx, dxp, pos, idx, map, k, S, d};
  if (k == 1) launch_gemm<kModeGateDx, 256, false, true, EpiGateDx<1>>(ta, tb, p, ep, 0, s);
  else if (k == 2) launch_gemm<kModeGateDx, 256, false, true, EpiGateDx<2>>(ta, tb, p, ep, 0, s);
  else launch_gemm<kModeGateDx, 256, false, true, EpiGateDx<0>>(ta, tb, p, ep, 0, s);
}

}  // namespace tamoe
