// Expert FFN as tcgen05 grouped GEMMs over the padded, expert-sorted token
// buffer produced by the permute kernel.
//
// Replaces the reference's inline linear expert (trainer.cpp:284-289 forward,
// trainer.cpp:310-316 expert gradient) and generalises it to the GPT-MoE
// two-layer FFN (d -> f -> d, GELU) the north-star configs name.
//
// Layouts (bf16, row-major):
//   tokens  [R x K]     R = padded rows, group g owns rows [seg_start[g], +seg_rows[g])
//   W_fwd   [G x M x K] forward weight of group g as M x K (K-major A)
//   out     [R x M]
// Forward / dgrad use "tokens on N" (swap-AB) tiles so a group's N extent is
// its token count rounded to 16 (not 128): weights are the M=128 operand.
#include <cuda_bf16.h>

#include "common.hpp"
#include "expert.hpp"
#include "gemm_sm100.cuh"
#include "gemm_launch.cuh"
#include "tma_host.hpp"

namespace tamoe {

__device__ __forceinline__ float act_fwd(int act, float x) {
  if (act == kActGelu) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float t = tanhf(k0 * (x + k1 * x * x * x));
    return 0.5f * x * (1.f + t);
  } else if (act == kActRelu) {
    return x > 0.f ? x : 0.f;
  }
  return x;
}

__device__ __forceinline__ float act_grad(int act, float x) {
  if (act == kActGelu) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float u = k0 * (x + k1 * x * x * x);
    const float t = tanhf(u);
    return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
  } else if (act == kActRelu) {
    return x > 0.f ? 1.f : 0.f;
  }
  return 1.f;
}

// ---------------------------------------------------------------- swap-AB epilogue
// acc[lane = weight row m][col = token c]  ->  out[token row][m]
struct EpiSwap {
  struct Params {
    __nv_bfloat16* out;      // [R x ld]
    __nv_bfloat16* pre_out;  // optional: pre-activation store (forward)
    const __nv_bfloat16* pre_in;  // optional: pre-activation for act' (dgrad)
    int ld;
    int act_out;   // activation applied on store (forward)
    int act_grad;  // activation derivative multiplied in (dgrad)
  };
  static __device__ __forceinline__ void run(const Params& e, const GemmParams& p, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int lane) {
    const int m = ti.m0 + q * 32 + lane;
    const int row0 = p.seg_start[ti.g] + ti.n0;
    for (int c0 = 0; c0 < ti.n; c0 += 32) {
      float v[32];
      load_acc32(tmem_tile, c0, v);
      const int cn = min(32, ti.n - c0);
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        if (c >= cn) break;
        const size_t off = static_cast<size_t>(row0 + c0 + c) * e.ld + m;
        float x = v[c];
        if (e.pre_in) x *= act_grad(e.act_grad, __bfloat162float(e.pre_in[off]));
        if (e.pre_out) e.pre_out[off] = __float2bfloat16(x);
        e.out[off] = __float2bfloat16(act_fwd(e.act_out, x));
      }
    }
  }
};

// ---------------------------------------------------------------- wgrad epilogue
// acc[lane = row m][col = n]  ->  out[g][m][n]  (zeros for empty groups)
struct EpiWgrad {
  struct Params {
    __nv_bfloat16* out;  // [G x Mw x Nw]
  };
  static __device__ __forceinline__ void run(const Params& e, const GemmParams& p, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int lane) {
    const int m = ti.m0 + q * 32 + lane;
    __nv_bfloat16* dst = e.out + (static_cast<size_t>(ti.g) * p.Mw + m) * p.Nw + ti.n0;
    for (int c0 = 0; c0 < ti.n; c0 += 32) {
      float v[32];
      if (ti.k_len > 0) {
        load_acc32(tmem_tile, c0, v);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 pk;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[8 * j + 0], v[8 * j + 1]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
        pk.x = *reinterpret_cast<uint32_t*>(&h0);
        pk.y = *reinterpret_cast<uint32_t*>(&h1);
        pk.z = *reinterpret_cast<uint32_t*>(&h2);
        pk.w = *reinterpret_cast<uint32_t*>(&h3);
        *reinterpret_cast<uint4*>(dst + c0 + 8 * j) = pk;
      }
    }
  }
};

static void check_groups(int G) { require(G >= 1 && G <= kMaxGroups, "group count out of range [1, 1024]"); }

void grouped_fwd(const __nv_bfloat16* tokens, const __nv_bfloat16* w, int G, int M, int K, int R,
                 const int* seg_start, const int* seg_rows, __nv_bfloat16* out, __nv_bfloat16* pre_out, int act,
                 cudaStream_t s) {
  check_groups(G);
  require(M % kBM == 0, "grouped_fwd: M must be a multiple of 128");
  require(K % 64 == 0, "grouped_fwd: K must be a multiple of 64");
  CUtensorMap ta = make_tmap_bf16(w, K, static_cast<uint64_t>(G) * M, K, kBM);
  CUtensorMap tb = make_tmap_bf16(tokens, K, R, K, 256);
  GemmParams p{G, seg_start, seg_rows, M, 0, K, 1, 1, 1, 1};
  EpiSwap::Params ep{out, pre_out, nullptr, M, act, kActNone};
  launch_gemm<kModeSwap, 256, false, false, EpiSwap>(ta, tb, p, ep, 0, s);
}

void grouped_dgrad(const __nv_bfloat16* grad_tokens, const __nv_bfloat16* w, int G, int M, int K, int R,
                   const int* seg_start, const int* seg_rows, __nv_bfloat16* out, const __nv_bfloat16* pre_in,
                   int act, cudaStream_t s) {
  // out[R x M] = grad_tokens[R x K] . W_g[K x M]  (W_g stored K x M: MN-major A operand)
  check_groups(G);
  require(M % kBM == 0, "grouped_dgrad: M must be a multiple of 128");
  require(K % 64 == 0, "grouped_dgrad: K must be a multiple of 64");
  CUtensorMap ta = make_tmap_bf16(w, M, static_cast<uint64_t>(G) * K, M, 64);
  CUtensorMap tb = make_tmap_bf16(grad_tokens, K, R, K, 256);
  GemmParams p{G, seg_start, seg_rows, M, 0, K, 1, 1, 1, 1};
  EpiSwap::Params ep{out, nullptr, pre_in, M, kActNone, pre_in ? act : kActNone};
  launch_gemm<kModeSwap, 256, true, false, EpiSwap>(ta, tb, p, ep, 0, s);
}

void grouped_wgrad(const __nv_bfloat16* a_tokens, const __nv_bfloat16* b_tokens, int G, int M, int N, int R,
                   const int* seg_start, const int* seg_rows, __nv_bfloat16* out, cudaStream_t s) {
  // out[g][M x N] = a_tokens[seg_g]^T . b_tokens[seg_g]
  check_groups(G);
  require(M % kBM == 0, "grouped_wgrad: M must be a multiple of 128");
  require(N % 256 == 0, "grouped_wgrad: N must be a multiple of 256");
  CUtensorMap ta = make_tmap_bf16(a_tokens, M, R, M, 64);
  CUtensorMap tb = make_tmap_bf16(b_tokens, N, R, N, 64);
  GemmParams p{G, seg_start, seg_rows, M, N, 0, 1, 1, 1, 1};
  EpiWgrad::Params ep{out};
  launch_gemm<kModeWgrad, 256, true, true, EpiWgrad>(ta, tb, p, ep, 0, s);
}

}  // namespace tamoe
