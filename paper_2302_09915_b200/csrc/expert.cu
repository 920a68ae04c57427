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

#include <cstdlib>
#include <type_traits>

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

// act(x) and act'(x) from one tanh
__device__ __forceinline__ void act_both(int act, float x, float& y, float& dy) {
  if (act == kActGelu) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float t = ptx::tanh_fast(k0 * (x + k1 * x * x * x));
    y = 0.5f * x * (1.f + t);
    dy = 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
  } else if (act == kActRelu) {
    y = x > 0.f ? x : 0.f;
    dy = x > 0.f ? 1.f : 0.f;
  } else {
    y = x;
    dy = 1.f;
  }
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
// Per epilogue warp (32 features, every other 32-token chunk): tcgen05.ld -> (x act'(pre), prefetched with
// cp.async two chunks ahead, starting before the accumulator is ready) -> bf16 staging tile
// [32 tokens][32 features] in smem -> one TMA bulk store.
struct SwapParams {
  CUtensorMap out32, out16;  // store maps of `out`: box {32 features, 32 | 16 tokens}
  CUtensorMap pre32, pre16;  // store maps of `pre_out`
  const __nv_bfloat16* pre_in;  // pre-activation for act' (dgrad)
  SwapPush push;                 // V = 3: peer destination of every output row
  int ld;
  int act_out;   // activation applied on store (forward)
  int act_grad;  // activation derivative multiplied in (dgrad)
};

// V = 0: plain store; 1: store act(x) and the activation derivative act'(x) (kept for the backward in
// place of the pre-activation); 2: multiply by the stored act'(x); 3: plain, each row stored into its
// home rank over NVLink (16-byte peer stores from the staging tile, 4 per lane and chunk).
//
// The transpose (accumulator rows = features, output rows = tokens) is done by the shared-memory store: the
// accumulator is read from TMEM in the mma fragment layout (tcgen05.ld 16x256b) and written with
// stmatrix.trans, four 8x8 tiles per instruction, into a staging tile [32 tokens][32 features] whose 16-byte
// pieces are XOR-swizzled by (token >> 1) & 3 -- the TMA 64-byte swizzle of the store maps, which makes the
// stmatrix rows (64 B apart) bank-conflict free.
__device__ __forceinline__ int swz64(int row, int piece) { return row * 32 + ((piece ^ ((row >> 1) & 3)) << 3); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_bf16x2(uint32_t v) {
  return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&v));
}

template <int V>
struct EpiSwap {
  static constexpr int kChunk = 2048;  // 32 x 32 bf16
  static constexpr int kPf = 2;        // own chunks of pre_in in flight
  // staging per warp: V0/V3 a 2-slot output ring; V1 2-slot rings for act(x) and act'(x) (4 pipeline stages:
  // single slots measured slower); V2 one output slot + the 2-slot act' prefetch ring (keeps 5 stages)
  static constexpr bool kRing = V != 2;
  static constexpr int kWarpBytes = (V == 1 ? 4 : (V == 2 ? 3 : 2)) * kChunk;
  static constexpr bool kEarlyRelease = true;
  static constexpr int kMaxCh = 4;  // a warp's chunks per tile: every other 32-column chunk of N <= 256
  using Params = SwapParams;
  static __device__ __forceinline__ void load_chunk(const Params& e, const TileInfo& ti, int row0, int mcol, int ch,
                                                    __nv_bfloat16* slot, int lane) {
    const int nch = (ti.n + 31) / 32;
    if (ch < nch) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int vid = lane + 32 * i;
        const int r = vid >> 2, part = vid & 3;
        const bool ok = ch * 32 + r < ti.n;
        const __nv_bfloat16* src =
            e.pre_in + static_cast<long long>(row0 + ch * 32 + (ok ? r : 0)) * e.ld + mcol + part * 8;
        ptx::cp_async_16(slot + swz64(r, part), src, ok);
      }
    }
    ptx::cp_async_commit();  // uniform group count, even when empty
  }
  static __device__ __forceinline__ void prefetch(const Params& e, const GemmParams&, const TileInfo& ti, int q, int h,
                                                  int lane, uint8_t* wsm, const int* s_start) {
    if constexpr (V == 2) {
      __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(wsm + kChunk);
      const int row0 = s_start[ti.g] + ti.n0;
      const int mcol = ti.m0 + q * 32;
      for (int j = 0; j < kPf; ++j) load_chunk(e, ti, row0, mcol, h + 2 * j, ring + j * 1024, lane);
    }
  }
  template <class Release>
  static __device__ __forceinline__ void run(const Params& e, const GemmParams&, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int h, int lane, uint8_t* wsm,
                                             const int* s_start, Release&& release) {
    // copy this warp's share of the accumulator to registers (fragment layout: acc[j][16 hh + 4 k + 2 rg + b] =
    // feature 16 hh + 8 rg + lane / 4, token 32 ch + 8 k + 2 (lane % 4) + b) and hand TMEM back at once
    const int nch_all = (ti.n + 31) / 32;
    uint32_t acc[kMaxCh][32];
#pragma unroll
    for (int j = 0; j < kMaxCh; ++j) {
      if (h + 2 * j < nch_all) {
        uint32_t r[16];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          ptx::tmem_ld_16x256b_x4(tmem_tile + (static_cast<uint32_t>(16 * hh) << 16) + (h + 2 * j) * 32, r);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[j][16 * hh + i] = r[i];
        }
      }
    }
    ptx::tmem_ld_wait();
    release();
    __nv_bfloat16* st_out = reinterpret_cast<__nv_bfloat16*>(wsm);
    __nv_bfloat16* extra = reinterpret_cast<__nv_bfloat16*>(wsm + (V == 1 ? 2 : 1) * kChunk);  // act' ring (V1 / V2)
    const int mcol = ti.m0 + q * 32;
    const int row0 = s_start[ti.g] + ti.n0;
    const int nch = (ti.n + 31) / 32;
    // this lane's stmatrix / ldmatrix row: token 8k + (lane % 8) of matrix (feature block) lane / 8
    const int srow = lane & 7, spiece = lane >> 3;
    if (lane == 0) ptx::bulk_wait_read<0>();  // staging tiles free again
    __syncwarp();
#pragma unroll
    for (int j = 0; j < kMaxCh; ++j) {
      const int ch = h + 2 * j;
      if (ch >= nch) break;
      if constexpr (V == 2) {
        ptx::cp_async_wait<kPf - 1>();
        __syncwarp();
      }
      if (kRing ? j >= 2 : j >= 1) {  // the slot's previous TMA store has read it
        if (lane == 0) {
          if constexpr (kRing) ptx::bulk_wait_read<1>();
          else ptx::bulk_wait_read<0>();
        }
        __syncwarp();
      }
      __nv_bfloat16* so = st_out + (kRing ? (j & 1) * 1024 : 0);
      __nv_bfloat16* sx = extra + (j & 1) * 1024;
      const uint32_t so_u = ptx::smem_u32(so), sx_u = ptx::smem_u32(sx);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t off = static_cast<uint32_t>(swz64(8 * k + srow, spiece)) * 2;
        uint32_t o[4], dy[4];
        if constexpr (V == 2) ptx::ldmatrix_x4_trans(sx_u + off, dy);
#pragma unroll
        for (int m = 0; m < 4; ++m) {  // matrix m = features 8m..8m+7 = (hh, rg) = (m >> 1, m & 1)
          const float x0 = __uint_as_float(acc[j][16 * (m >> 1) + 4 * k + 2 * (m & 1)]);
          const float x1 = __uint_as_float(acc[j][16 * (m >> 1) + 4 * k + 2 * (m & 1) + 1]);
          if constexpr (V == 1) {
            float y0, y1, d0, d1;
            act_both(e.act_out, x0, y0, d0);
            act_both(e.act_out, x1, y1, d1);
            o[m] = pack_bf16x2(y0, y1);
            dy[m] = pack_bf16x2(d0, d1);
          } else if constexpr (V == 2) {
            const float2 g = unpack_bf16x2(dy[m]);
            o[m] = pack_bf16x2(x0 * g.x, x1 * g.y);
          } else {  // V = 0 / 3
            o[m] = pack_bf16x2(act_fwd(e.act_out, x0), act_fwd(e.act_out, x1));
          }
        }
        ptx::stmatrix_x4_trans(so_u + off, o[0], o[1], o[2], o[3]);
        if constexpr (V == 1) ptx::stmatrix_x4_trans(sx_u + off, dy[0], dy[1], dy[2], dy[3]);
      }
      if constexpr (V == 3) {
        __syncwarp();
        const int rows = min(32, ti.n - ch * 32);
        const int y = row0 + ch * 32;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = (lane >> 2) + 8 * i;
          if (r < rows) {
            const int code = __ldg(e.push.row_code + y + r);
            const uint4 v = *reinterpret_cast<const uint4*>(so + swz64(r, lane & 3));
            __nv_bfloat16* dst = e.push.dst.p[code >> kPushRowBits] +
                                 static_cast<long long>(code & ((1 << kPushRowBits) - 1)) * e.ld + mcol + (lane & 3) * 8;
            *reinterpret_cast<uint4*>(dst) = v;
            const int rep = e.push.dst.rep[code >> kPushRowBits];
            if (rep > 1) store_repeat(dst, v, rep);
          }
        }
        __syncwarp();  // staging slot free again
        continue;
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if constexpr (V == 2) load_chunk(e, ti, row0, mcol, ch + 2 * kPf, sx, lane);  // refill the consumed slot
      if (lane == 0) {
        const int rows = min(32, ti.n - ch * 32);
        const int y = row0 + ch * 32;
        ptx::tma_store_2d(rows == 32 ? &e.out32 : &e.out16, so, mcol, y);
        if constexpr (V == 1) ptx::tma_store_2d(rows == 32 ? &e.pre32 : &e.pre16, sx, mcol, y);
        ptx::bulk_commit();
      }
    }
    if constexpr (V == 2) ptx::cp_async_wait<0>();
    __syncwarp();
  }
  static __device__ __forceinline__ void finish(const Params&, int lane) {
    if (lane == 0) ptx::bulk_wait<0>();
    if constexpr (V == 3) __threadfence_system();  // pushed rows visible before the phase barrier signals
    __syncwarp();
  }
};

// ---------------------------------------------------------------- wgrad epilogue
// acc[lane = row m][col = n]  ->  out[g][m][n]  (zeros for empty groups).  Per warp and 32-column
// chunk (every other chunk): bf16 staging tile [32 rows][32 cols] in the TMA 64-byte swizzle layout,
// one bulk store.
struct EpiWgrad {
  static constexpr int kWarpBytes = 2 * 2048;
  static constexpr bool kEarlyRelease = true;
  struct Params {
    CUtensorMap out;  // [G*Mw x Nw], box {32, 32}, 64B swizzle
  };
  static __device__ __forceinline__ void prefetch(const Params&, const GemmParams&, const TileInfo&, int, int, int,
                                                  uint8_t*, const int*) {}
  template <class Release>
  static __device__ __forceinline__ void run(const Params& e, const GemmParams& p, const TileInfo& ti,
                                             uint32_t tmem_tile, int q, int h, int lane, uint8_t* wsm, const int*,
                                             Release&& release) {
    // BN = 256: four 32-column chunks per warp, copied out of TMEM before any math / store
    float acc[4][32];
    if (ti.k_len > 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem_tile + 32 * h + 64 * j, r);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[j][i] = __uint_as_float(r[i]);
      }
      ptx::tmem_ld_wait();
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[j][i] = 0.f;
    }
    release();
    if (lane == 0) ptx::bulk_wait_read<0>();
    __syncwarp();
    const int row = ti.g * p.Mw + ti.m0 + q * 32;
    const int sw = (lane >> 1) & 3;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c0 = 32 * h + 64 * j;
      const float* v = acc[j];
      if (j >= 2) {
        if (lane == 0) ptx::bulk_wait_read<1>();
        __syncwarp();
      }
      uint8_t* st = wsm + (j & 1) * 2048 + lane * 64;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        uint4 pk;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[8 * jj + 0], v[8 * jj + 1]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(v[8 * jj + 2], v[8 * jj + 3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * jj + 4], v[8 * jj + 5]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(v[8 * jj + 6], v[8 * jj + 7]);
        pk.x = *reinterpret_cast<uint32_t*>(&h0);
        pk.y = *reinterpret_cast<uint32_t*>(&h1);
        pk.z = *reinterpret_cast<uint32_t*>(&h2);
        pk.w = *reinterpret_cast<uint32_t*>(&h3);
        *reinterpret_cast<uint4*>(st + ((jj ^ sw) * 16)) = pk;
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_2d(&e.out, wsm + (j & 1) * 2048, ti.n0 + c0, row);
        ptx::bulk_commit();
      }
    }
  }
  static __device__ __forceinline__ void finish(const Params&, int lane) {
    if (lane == 0) ptx::bulk_wait<0>();
    __syncwarp();
  }
};

// ---------------------------------------------------------------- chained swap GEMMs
// Two swap GEMMs in one persistent launch (GemmParams::chain): tiles of the first use E0, tiles of the second E1 and
// the second's tensor maps.  FFN forward: fwd1 (E0 = act + act' out) -> fwd2 (E1 = plain / pushed output); FFN
// backward: dgrad2 (E0 = x act') -> dgrad1 (E1).
template <class E0, class E1>
struct EpiChain {
  static constexpr bool kChained = true;
  static constexpr bool kEarlyRelease = true;
  static_assert(E0::kEarlyRelease && E1::kEarlyRelease, "chained epilogues release TMEM early");
  static constexpr int kWarpBytes = E0::kWarpBytes > E1::kWarpBytes ? E0::kWarpBytes : E1::kWarpBytes;
  struct Params {
    typename E0::Params p0;
    typename E1::Params p1;
    CUtensorMap tmA2, tmB2;  // the second GEMM's operands
  };
  // the engine runs the two phases' tiles in two consecutive epilogue loops (a CTA's first-GEMM tiles all precede
  // its second-GEMM tiles), so each loop inlines only its own epilogue body
  using First = E0;
  using Second = E1;
  static __device__ __forceinline__ const typename E0::Params& params(const Params& e, std::integral_constant<int, 0>) {
    return e.p0;
  }
  static __device__ __forceinline__ const typename E1::Params& params(const Params& e, std::integral_constant<int, 1>) {
    return e.p1;
  }
};

// cg: CTAs per cluster -- 1, 2 (a pair: cta_group::2, M = 256) or 4 (two pairs on adjacent 256-row weight blocks
// sharing the token operand by TMA multicast)
template <int kMode, int BN, bool A_MN, bool B_MN, class Epi>
static void launch_pair_or_single(int cg, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                                  const typename Epi::Params& ep, cudaStream_t s) {
  if constexpr (kMode == kModeSwap && !B_MN) {
    if (cg == 4) {
      launch_gemm<kMode, BN, A_MN, B_MN, Epi, 4>(ta, tb, p, ep, 0, s);
      return;
    }
  }
  if (cg >= 2) launch_gemm<kMode, BN, A_MN, B_MN, Epi, 2>(ta, tb, p, ep, 0, s);
  else launch_gemm<kMode, BN, A_MN, B_MN, Epi, 1>(ta, tb, p, ep, 0, s);
}

// Swap-GEMM cluster shape for M weight rows: one pair when M % 256 == 0, else single CTAs.  TAMOE_MC=1 selects
// two multicasting pairs when M % 512 == 0 -- correct, but measured 3-18 % slower at C2, so off.
static int swap_cluster(int M) {
  static const int mc = [] {
    const char* v = std::getenv("TAMOE_MC");
    return v ? std::atoi(v) : 0;
  }();
  if (M % 512 == 0 && mc) return 4;
  return M % 256 == 0 ? 2 : 1;
}

static uint32_t swap_token_box(int cg) { return cg == 4 ? 64 : (cg == 2 ? 128 : 256); }

static SwapParams swap_params(__nv_bfloat16* out, __nv_bfloat16* pre_out, const __nv_bfloat16* pre_in, int M,
                              int R, int act_out, int act_grad) {
  SwapParams e;
  // staging tiles are 64-byte swizzled (EpiSwap: conflict-free stmatrix rows)
  e.out32 = make_tmap_bf16_box(out, M, R, M, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  e.out16 = make_tmap_bf16_box(out, M, R, M, 32, 16, CU_TENSOR_MAP_SWIZZLE_64B);
  if (pre_out) {
    e.pre32 = make_tmap_bf16_box(pre_out, M, R, M, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    e.pre16 = make_tmap_bf16_box(pre_out, M, R, M, 32, 16, CU_TENSOR_MAP_SWIZZLE_64B);
  } else {
    e.pre32 = e.out32;
    e.pre16 = e.out16;
  }
  e.pre_in = pre_in;
  e.ld = M;
  e.act_out = act_out;
  e.act_grad = act_grad;
  return e;
}




static void check_groups(int G) { require(G >= 1 && G <= kMaxGroups, "group count out of range [1, 256]"); }


void grouped_fwd(const __nv_bfloat16* tokens, const __nv_bfloat16* w, int G, int M, int K, int R,
                 const int* seg_start, const int* seg_rows, __nv_bfloat16* out, __nv_bfloat16* pre_out, int act,
                 cudaStream_t s, int w_mod, const SwapPush* push) {
  check_groups(G);
  require(M % kBM == 0, "grouped_fwd: M must be a multiple of 128");
  require(K % 64 == 0, "grouped_fwd: K must be a multiple of 64");
  const int pair = swap_cluster(M);
  const int Gw = w_mod > 0 ? w_mod : G;  // distinct weight matrices
  CUtensorMap ta = make_tmap_bf16(w, K, static_cast<uint64_t>(Gw) * M, K, kBM);
  CUtensorMap tb = make_tmap_bf16(tokens, K, R, K, swap_token_box(pair));
  GemmParams p{G, seg_start, seg_rows, M, 0, K, 1, 1, 1, 1, w_mod, 1};
  SwapParams ep = swap_params(out, pre_out, nullptr, M, R, act, kActNone);
  require(!(push && pre_out), "grouped_fwd: push needs a plain output");
  if (push) {
    ep.push = *push;
    launch_pair_or_single<kModeSwap, 256, false, false, EpiSwap<3>>(pair, ta, tb, p, ep, s);
  } else if (pre_out) {
    launch_pair_or_single<kModeSwap, 256, false, false, EpiSwap<1>>(pair, ta, tb, p, ep, s);
  } else {
    launch_pair_or_single<kModeSwap, 256, false, false, EpiSwap<0>>(pair, ta, tb, p, ep, s);
  }
}

void grouped_dgrad(const __nv_bfloat16* grad_tokens, const __nv_bfloat16* w, int G, int M, int K, int R,
                   const int* seg_start, const int* seg_rows, __nv_bfloat16* out, const __nv_bfloat16* pre_in,
                   int act, cudaStream_t s, int w_mod, const SwapPush* push) {
  // out[R x M] = grad_tokens[R x K] . W_g[K x M]  (W_g stored K x M: MN-major A operand)
  check_groups(G);
  require(M % kBM == 0, "grouped_dgrad: M must be a multiple of 128");
  require(K % 64 == 0, "grouped_dgrad: K must be a multiple of 64");
  const int pair = swap_cluster(M);
  const int Gw = w_mod > 0 ? w_mod : G;
  CUtensorMap ta = make_tmap_bf16(w, M, static_cast<uint64_t>(Gw) * K, M, 64);
  CUtensorMap tb = make_tmap_bf16(grad_tokens, K, R, K, swap_token_box(pair));
  GemmParams p{G, seg_start, seg_rows, M, 0, K, 1, 1, 1, 1, w_mod, 1};
  SwapParams ep = swap_params(out, nullptr, pre_in, M, R, kActNone, pre_in ? act : kActNone);
  require(!(push && pre_in), "grouped_dgrad: push needs a plain output");
  if (push) {
    ep.push = *push;
    launch_pair_or_single<kModeSwap, 256, true, false, EpiSwap<3>>(pair, ta, tb, p, ep, s);
  } else if (pre_in) {
    launch_pair_or_single<kModeSwap, 256, true, false, EpiSwap<2>>(pair, ta, tb, p, ep, s);
  } else {
    launch_pair_or_single<kModeSwap, 256, true, false, EpiSwap<0>>(pair, ta, tb, p, ep, s);
  }
}

void grouped_wgrad(const __nv_bfloat16* a_tokens, const __nv_bfloat16* b_tokens, int G, int M, int N, int R,
                   const int* seg_start, const int* seg_rows, __nv_bfloat16* out, cudaStream_t s, int nsub) {
  // out[g][M x N] = a_tokens[seg_g]^T . b_tokens[seg_g]
  check_groups(G);
  require(M % kBM == 0, "grouped_wgrad: M must be a multiple of 128");
  require(N % 256 == 0, "grouped_wgrad: N must be a multiple of 256");
  CUtensorMap ta = make_tmap_bf16(a_tokens, M, R, M, 64);
  CUtensorMap tb = make_tmap_bf16(b_tokens, N, R, N, 64);
  require(nsub >= 1 && G * nsub <= kMaxGroups, "grouped_wgrad: too many sub-segments");
  GemmParams p{G, seg_start, seg_rows, M, N, 0, 1, 1, 1, 1, 0, nsub};
  EpiWgrad::Params ep{make_tmap_bf16_box(out, N, static_cast<uint64_t>(G) * M, N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)};
  launch_pair_or_single<kModeWgrad, 256, true, true, EpiWgrad>(M % 256 == 0 ? 2 : 1, ta, tb, p, ep, s);
}

static void chain_params(GemmParams& p, int M2, int K2, int* ready, int stride, int M1) {
  p.chain = 1;
  p.Mw2 = M2;
  p.Kw2 = K2;
  p.ready = ready;
  p.ready_stride = stride;
  // every epilogue warp of both CTAs of every first-GEMM m block signals once per (group, token tile)
  p.ready_target = (M1 / 256) * kEpiWarps * 2;
}

int chain_ready_stride(int R) { return (R + 255) / 256 + 1; }

void grouped_ffn_fwd_chain(const __nv_bfloat16* tokens, const __nv_bfloat16* w1, const __nv_bfloat16* w2, int G,
                           int f, int d, int d_out, int R, const int* seg_start, const int* seg_rows,
                           __nv_bfloat16* H, __nv_bfloat16* dact, __nv_bfloat16* out, int act, int* ready,
                           cudaStream_t s, int w_mod, const SwapPush* push) {
  check_groups(G);
  require(f % 256 == 0 && d_out % 256 == 0 && d % 64 == 0 && f % 64 == 0, "chained FFN forward: f, d_out % 256");
  const int Gw = w_mod > 0 ? w_mod : G;
  CUtensorMap ta = make_tmap_bf16(w1, d, static_cast<uint64_t>(Gw) * f, d, kBM);
  CUtensorMap tb = make_tmap_bf16(tokens, d, R, d, swap_token_box(2));
  GemmParams p{G, seg_start, seg_rows, f, 0, d, 1, 1, 1, 1, w_mod, 1};
  const int stride = chain_ready_stride(R);
  chain_params(p, d_out, f, ready, stride, f);
  TAMOE_CUDA(cudaMemsetAsync(ready, 0, sizeof(int) * static_cast<size_t>(G) * stride, s));
  if (push) {
    EpiChain<EpiSwap<1>, EpiSwap<3>>::Params ep{swap_params(H, dact, nullptr, f, R, act, kActNone),
                                                swap_params(out, nullptr, nullptr, d_out, R, kActNone, kActNone),
                                                make_tmap_bf16(w2, f, static_cast<uint64_t>(Gw) * d_out, f, kBM),
                                                make_tmap_bf16(H, f, R, f, swap_token_box(2))};
    ep.p1.push = *push;
    launch_gemm<kModeSwap, 256, false, false, EpiChain<EpiSwap<1>, EpiSwap<3>>, 2>(ta, tb, p, ep, 0, s);
  } else {
    EpiChain<EpiSwap<1>, EpiSwap<0>>::Params ep{swap_params(H, dact, nullptr, f, R, act, kActNone),
                                                swap_params(out, nullptr, nullptr, d_out, R, kActNone, kActNone),
                                                make_tmap_bf16(w2, f, static_cast<uint64_t>(Gw) * d_out, f, kBM),
                                                make_tmap_bf16(H, f, R, f, swap_token_box(2))};
    launch_gemm<kModeSwap, 256, false, false, EpiChain<EpiSwap<1>, EpiSwap<0>>, 2>(ta, tb, p, ep, 0, s);
  }
}

void grouped_ffn_dgrad_chain(const __nv_bfloat16* dO, const __nv_bfloat16* w2, const __nv_bfloat16* w1, int G, int f,
                             int d, int d_out, int R, const int* seg_start, const int* seg_rows, __nv_bfloat16* dA,
                             const __nv_bfloat16* dact, __nv_bfloat16* dx_out, int act, int* ready, cudaStream_t s,
                             int w_mod, const SwapPush* push) {
  // dA[R x f] = (dO[R x d_out] . W2_g) * act';  dx[R x d] = dA . W1_g   (W2_g stored d_out x f, W1_g f x d: MN-major A)
  check_groups(G);
  require(f % 256 == 0 && d % 256 == 0 && d_out % 64 == 0 && f % 64 == 0, "chained FFN dgrad: f, d % 256");
  const int Gw = w_mod > 0 ? w_mod : G;
  CUtensorMap ta = make_tmap_bf16(w2, f, static_cast<uint64_t>(Gw) * d_out, f, 64);
  CUtensorMap tb = make_tmap_bf16(dO, d_out, R, d_out, swap_token_box(2));
  GemmParams p{G, seg_start, seg_rows, f, 0, d_out, 1, 1, 1, 1, w_mod, 1};
  const int stride = chain_ready_stride(R);
  chain_params(p, d, f, ready, stride, f);
  TAMOE_CUDA(cudaMemsetAsync(ready, 0, sizeof(int) * static_cast<size_t>(G) * stride, s));
  if (push) {
    EpiChain<EpiSwap<2>, EpiSwap<3>>::Params ep{swap_params(dA, nullptr, dact, f, R, kActNone, act),
                                                swap_params(dx_out, nullptr, nullptr, d, R, kActNone, kActNone),
                                                make_tmap_bf16(w1, d, static_cast<uint64_t>(Gw) * f, d, 64),
                                                make_tmap_bf16(dA, f, R, f, swap_token_box(2))};
    ep.p1.push = *push;
    launch_gemm<kModeSwap, 256, true, false, EpiChain<EpiSwap<2>, EpiSwap<3>>, 2>(ta, tb, p, ep, 0, s);
  } else {
    EpiChain<EpiSwap<2>, EpiSwap<0>>::Params ep{swap_params(dA, nullptr, dact, f, R, kActNone, act),
                                                swap_params(dx_out, nullptr, nullptr, d, R, kActNone, kActNone),
                                                make_tmap_bf16(w1, d, static_cast<uint64_t>(Gw) * f, d, 64),
                                                make_tmap_bf16(dA, f, R, f, swap_token_box(2))};
    launch_gemm<kModeSwap, 256, true, false, EpiChain<EpiSwap<2>, EpiSwap<0>>, 2>(ta, tb, p, ep, 0, s);
  }
}

}  // namespace tamoe
