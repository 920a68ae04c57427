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
    const float t = ptx::tanh_fast(k0 * (x + k1 * x * x * x));
    return 0.5f * x * (1.f + t);
  } else if (act == kActRelu) {
    return x > 0.f ? x : 0.f;
  }
  return x;
}

__device__ __forceinline__ float act_grad(int act, float x) {
  if (act == kActGelu) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float t = ptx::tanh_fast(k0 * (x + k1 * x * x * x));
    return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
  } else if (act == kActRelu) {
    return x > 0.f ? 1.f : 0.f;
  }
  return 1.f;
}

// ---------------------------------------------------------------- swap-AB epilogue
// acc[lane = weight row m][col = token c]  ->  out[token row][m]
// Per epilogue warp (32 features) and 32-token chunk: tcgen05.ld -> (x act'(pre), prefetched with
// cp.async) -> bf16 staging tile [32 tokens][32 features] in smem -> one TMA bulk store.
struct EpiSwap {
  static constexpr int kChunk = 2048;            // 32 x 32 bf16
  static constexpr int kWarpBytes = 6 * kChunk;  // out x2, pre_out x2, pre_in prefetch x2
  static constexpr int kSmemBytes = 4 * kWarpBytes;
  struct Params {
    CUtensorMap out32, out16;  // store maps of `out`: box {32 features, 32 | 16 tokens}
    CUtensorMap pre32, pre16;  // store maps of `pre_out`
    const __nv_bfloat16* pre_in;  // optional: pre-activation for act' (dgrad)
    int ld;
    int act_out;   // activation applied on store (forward)
    int act_grad;  // activation derivative multiplied in (dgrad)
    int has_pre_out;
  };
  static __device__ __forceinline__ void run(const Params& e, const GemmParams& p, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int lane, uint8_t* smem) {
    uint8_t* ws = smem + q * kWarpBytes;
    __nv_bfloat16* st_out = reinterpret_cast<__nv_bfloat16*>(ws);
    __nv_bfloat16* st_pre = reinterpret_cast<__nv_bfloat16*>(ws + 2 * kChunk);
    __nv_bfloat16* pf = reinterpret_cast<__nv_bfloat16*>(ws + 4 * kChunk);
    const int mcol = ti.m0 + q * 32;
    const int row0 = p.seg_start[ti.g] + ti.n0;
    const int nch = (ti.n + 31) / 32;
    const bool has_pre_in = e.pre_in != nullptr;
    // all earlier bulk stores of this warp must have finished reading the staging tiles
    if (lane == 0) ptx::bulk_wait_read<0>();
    __syncwarp();
    auto prefetch = [&](int ch) {
      __nv_bfloat16* dst = pf + (ch & 1) * 1024;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int vid = lane + 32 * i;
        const int r = vid >> 2, part = vid & 3;
        const bool ok = ch * 32 + r < ti.n;
        const __nv_bfloat16* src = e.pre_in + static_cast<long long>(row0 + ch * 32 + (ok ? r : 0)) * e.ld + mcol + part * 8;
        ptx::cp_async_16(dst + r * 32 + part * 8, src, ok);
      }
      ptx::cp_async_commit();
    };
    if (has_pre_in) prefetch(0);
    for (int ch = 0; ch < nch; ++ch) {
      const int buf = ch & 1;
      if (has_pre_in) {
        if (ch + 1 < nch) prefetch(ch + 1);
        else ptx::cp_async_commit();
        ptx::cp_async_wait<1>();
        __syncwarp();
      }
      float v[32];
      load_acc32(tmem_tile, ch * 32, v);
      if (ch >= 2) {
        if (lane == 0) ptx::bulk_wait_read<1>();
        __syncwarp();
      }
      __nv_bfloat16* so = st_out + buf * 1024;
      __nv_bfloat16* sp = st_pre + buf * 1024;
      const __nv_bfloat16* pin = pf + buf * 1024;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        float x = v[c];
        if (has_pre_in) x *= act_grad(e.act_grad, __bfloat162float(pin[c * 32 + lane]));
        if (e.has_pre_out) sp[c * 32 + lane] = __float2bfloat16(x);
        so[c * 32 + lane] = __float2bfloat16(act_fwd(e.act_out, x));
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int rows = min(32, ti.n - ch * 32);
        const int y = row0 + ch * 32;
        ptx::tma_store_2d(rows == 32 ? &e.out32 : &e.out16, so, mcol, y);
        if (e.has_pre_out) ptx::tma_store_2d(rows == 32 ? &e.pre32 : &e.pre16, sp, mcol, y);
        ptx::bulk_commit();
      }
    }
  }
  static __device__ __forceinline__ void finish(const Params&, int, int lane) {
    if (lane == 0) ptx::bulk_wait<0>();
    __syncwarp();
  }
};

// ---------------------------------------------------------------- wgrad epilogue
// acc[lane = row m][col = n]  ->  out[g][m][n]  (zeros for empty groups).  Per warp and 32-column
// chunk: bf16 staging tile [32 rows][32 cols] in the TMA 64-byte swizzle layout, one bulk store.
struct EpiWgrad {
  static constexpr int kWarpBytes = 2 * 2048;
  static constexpr int kSmemBytes = 4 * kWarpBytes;
  struct Params {
    CUtensorMap out;  // [G*Mw x Nw], box {32, 32}, 64B swizzle
  };
  static __device__ __forceinline__ void run(const Params& e, const GemmParams& p, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int lane, uint8_t* smem) {
    uint8_t* ws = smem + q * kWarpBytes;
    if (lane == 0) ptx::bulk_wait_read<0>();
    __syncwarp();
    const int row = ti.g * p.Mw + ti.m0 + q * 32;
    const int sw = (lane >> 1) & 3;
    for (int c0 = 0, ch = 0; c0 < ti.n; c0 += 32, ++ch) {
      float v[32];
      if (ti.k_len > 0) {
        load_acc32(tmem_tile, c0, v);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      if (ch >= 2) {
        if (lane == 0) ptx::bulk_wait_read<1>();
        __syncwarp();
      }
      uint8_t* st = ws + (ch & 1) * 2048 + lane * 64;
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
        *reinterpret_cast<uint4*>(st + ((j ^ sw) * 16)) = pk;
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_2d(&e.out, ws + (ch & 1) * 2048, ti.n0 + c0, row);
        ptx::bulk_commit();
      }
    }
  }
  static __device__ __forceinline__ void finish(const Params&, int, int lane) {
    if (lane == 0) ptx::bulk_wait<0>();
    __syncwarp();
  }
};

static EpiSwap::Params swap_params(__nv_bfloat16* out, __nv_bfloat16* pre_out, const __nv_bfloat16* pre_in, int M,
                                   int R, int act_out, int act_grad) {
  EpiSwap::Params e;
  e.out32 = make_tmap_bf16_box(out, M, R, M, 32, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
  e.out16 = make_tmap_bf16_box(out, M, R, M, 32, 16, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (pre_out) {
    e.pre32 = make_tmap_bf16_box(pre_out, M, R, M, 32, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    e.pre16 = make_tmap_bf16_box(pre_out, M, R, M, 32, 16, CU_TENSOR_MAP_SWIZZLE_NONE);
  } else {
    e.pre32 = e.out32;
    e.pre16 = e.out16;
  }
  e.pre_in = pre_in;
  e.ld = M;
  e.act_out = act_out;
  e.act_grad = act_grad;
  e.has_pre_out = pre_out != nullptr;
  return e;
}

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
  EpiSwap::Params ep = swap_params(out, pre_out, nullptr, M, R, act, kActNone);
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
  EpiSwap::Params ep = swap_params(out, nullptr, pre_in, M, R, kActNone, pre_in ? act : kActNone);
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
  EpiWgrad::Params ep{make_tmap_bf16_box(out, N, static_cast<uint64_t>(G) * M, N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)};
  launch_gemm<kModeWgrad, 256, true, true, EpiWgrad>(ta, tb, p, ep, 0, s);
}

}  // namespace tamoe
