// Persistent, warp-specialised tcgen05 GEMM engine shared by every dense
// contraction on the TA-MoE hot path (fused gate logits, expert FFN forward /
// dgrad / wgrad, gate dW and dX).
//
//   warps 0-3 : epilogue (warp q owns TMEM lanes 32q..32q+31)
//   warp 4    : TMA producer (one elected lane)
//   warp 5    : TMEM allocator + MMA issuer (one elected lane)
//
// A tile is always M=128 (TMEM lanes) x N<=BN (TMEM columns) x K (multiple of
// 16).  Operands are staged by TMA with 128-byte swizzle; each operand can be
// K-major (rows of 64 K-elements) or MN-major (64-element MN chunks of 64
// K-rows).  The fp32 accumulator is double buffered in TMEM so the epilogue of
// tile i overlaps the MMAs of tile i+1.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "ptx.cuh"

namespace tamoe {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kGemmThreads = 192;
constexpr int kMaxGroups = 1024;

enum GemmMode : int {
  kModeSwap = 0,    // M = weight rows (fixed), N = tokens of group g (variable), K fixed
  kModeWgrad = 1,   // M, N fixed, K = tokens of group g (variable)
  kModeGate = 2,    // M = tokens (all), N = experts (padded), K = d; weights per process
  kModeGateDw = 3,  // M = d, N = experts (64-multiple), K = tokens, split-K
  kModeGateDx = 4,  // M = tokens, N = d, K = experts (padded); weights per process
};

struct GemmParams {
  int num_groups;
  const int* seg_start;  // [G] first (padded) row of group g in the token buffers
  const int* seg_rows;   // [G] padded row count (multiple of 16)
  int Mw, Nw, Kw;        // see GemmMode
  int k_split;           // kModeGateDw: K splits per process
  int tokens_per_proc;   // rows per logical process (gate modes)
  int w_rows_per_proc;   // weight rows per process (gate modes)
  int procs;             // logical processes (gate modes)
};

struct TileInfo {
  int g;       // group
  int m0, n0;  // offsets within the group's output
  int n;       // valid N columns (multiple of 16, <= BN)
  int k_len;   // K extent (multiple of 16)
  int ks;      // split index (kModeGateDw)
  int ax, ay;  // A TMA base coordinates (see load_stage)
  int bx, by;  // B TMA base coordinates
};

// Epilogues may declare `static constexpr int kSmemBytes` of scratch shared memory (per CTA).
template <class Epi, class = void>
struct EpiSmem {
  static constexpr int value = 0;
};
template <class Epi>
struct EpiSmem<Epi, decltype(void(Epi::kSmemBytes))> {
  static constexpr int value = Epi::kSmemBytes;
};

template <int BN, int kEpiBytes = 0>
struct GemmSmem {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBudget = 220 * 1024 - kEpiBytes - 8 * 1024;
  static constexpr int kMaxStages = (BN >= 256) ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int kStages = (kBudget / kStageBytes < kMaxStages) ? kBudget / kStageBytes : kMaxStages;
  static_assert(kStages >= 2, "not enough shared memory for the pipeline");
  static constexpr int kEpiOffset = kStages * kStageBytes;
  static constexpr int kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr int kBarOffset = kEpiOffset + ((kEpiBytes + 1023) / 1024) * 1024;
  // barriers: full[S], empty[S], tfull[2], tempty[2]; tmem addr; tile prefix
  static constexpr int kMiscBytes = (2 * kStages + 4) * 8 + 16 + (kMaxGroups + 1) * 4;
  static constexpr int kTotal = kBarOffset + kMiscBytes + 1024;  // + alignment slack
};

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Number of tiles of group g (device side; prefix built once per CTA).
template <int kMode, int BN>
__device__ __forceinline__ int group_tiles(const GemmParams& p, int g) {
  if constexpr (kMode == kModeSwap) {
    return (p.Mw / kBM) * ceil_div(p.seg_rows[g], BN);
  } else if constexpr (kMode == kModeWgrad) {
    return (p.Mw / kBM) * (p.Nw / BN);
  } else if constexpr (kMode == kModeGate) {
    return p.procs * ceil_div(p.tokens_per_proc, kBM);
  } else if constexpr (kMode == kModeGateDw) {
    return p.procs * (p.Mw / kBM) * (p.Nw / BN) * p.k_split;
  } else {
    return p.procs * ceil_div(p.tokens_per_proc, kBM) * (p.Nw / BN);
  }
}

template <int kMode, int BN>
__device__ __forceinline__ void decode_tile(const GemmParams& p, const int* prefix, int t, TileInfo& ti) {
  // find group: prefix[g] <= t < prefix[g+1]
  int lo = 0, hi = p.num_groups - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const int g = lo;
  int r = t - prefix[g];
  ti.g = g;
  ti.ks = 0;
  if constexpr (kMode == kModeSwap) {
    const int rows = p.seg_rows[g];
    const int nb = ceil_div(rows, BN);
    const int mb = r / nb, nbk = r % nb;
    ti.m0 = mb * kBM;
    ti.n0 = nbk * BN;
    ti.n = min(BN, rows - ti.n0);
    ti.k_len = p.Kw;
    // A (weights): K-major -> (k, g*Mw + m0) ; MN-major -> (m0, g*Kw + k)
    ti.ax = 0; ti.ay = g * p.Mw + ti.m0;  // overwritten below for MN-major A by caller convention
    ti.bx = 0; ti.by = p.seg_start[g] + ti.n0;
  } else if constexpr (kMode == kModeWgrad) {
    const int nb = p.Nw / BN;
    ti.m0 = (r / nb) * kBM;
    ti.n0 = (r % nb) * BN;
    ti.n = BN;
    ti.k_len = p.seg_rows[g];
    ti.ax = ti.m0; ti.ay = p.seg_start[g];
    ti.bx = ti.n0; ti.by = p.seg_start[g];
  } else if constexpr (kMode == kModeGate) {
    // tile r -> (process, 128-token block); rows beyond the process' S are masked by the epilogue
    const int tb = ceil_div(p.tokens_per_proc, kBM);
    const int proc = r / tb;
    ti.g = proc;
    ti.m0 = (r % tb) * kBM;
    ti.n0 = 0;
    ti.n = BN;
    ti.k_len = p.Kw;
    ti.ax = 0; ti.ay = proc * p.tokens_per_proc + ti.m0;
    ti.bx = 0; ti.by = proc * p.w_rows_per_proc;
  } else if constexpr (kMode == kModeGateDw) {
    // tile r -> (process, split, m block, n block); K = the process' tokens
    const int nb = p.Nw / BN;
    const int per_split = (p.Mw / kBM) * nb;
    const int per_proc = per_split * p.k_split;
    const int proc = r / per_proc;
    const int rr0 = r % per_proc;
    ti.g = proc;
    ti.ks = rr0 / per_split;
    const int rr = rr0 % per_split;
    ti.m0 = (rr / nb) * kBM;
    ti.n0 = (rr % nb) * BN;
    ti.n = BN;
    const int chunk = ceil_div(ceil_div(p.tokens_per_proc, p.k_split), kBK) * kBK;
    const int kb = ti.ks * chunk;
    ti.k_len = max(0, min(p.tokens_per_proc, kb + chunk) - kb);
    ti.k_len = (ti.k_len + 15) & ~15;
    ti.ax = ti.m0; ti.ay = proc * p.tokens_per_proc + kb;
    ti.bx = ti.n0; ti.by = proc * p.tokens_per_proc + kb;
  } else {  // kModeGateDx: tile r -> (process, 128-token block, n block)
    const int nb = p.Nw / BN;
    const int tb = ceil_div(p.tokens_per_proc, kBM);
    const int proc = r / (tb * nb);
    const int rr = r % (tb * nb);
    ti.g = proc;
    ti.m0 = (rr / nb) * kBM;
    ti.n0 = (rr % nb) * BN;
    ti.n = BN;
    ti.k_len = p.Kw;
    ti.ax = 0; ti.ay = proc * p.tokens_per_proc + ti.m0;
    ti.bx = ti.n0; ti.by = proc * p.w_rows_per_proc;
  }
}

// Epilogue contract:
//   struct Epi { struct Params; static __device__ void run(const Params&, const GemmParams&,
//                const TileInfo&, uint32_t tmem_tile /*lane 0 col 0 of this tile*/, int q /*warp*/, int lane,
//                uint8_t* smem /*kSmemBytes scratch*/);
//                static __device__ void finish(const Params&, int q, int lane); };
template <int kMode, int BN, bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const GemmParams p, const __grid_constant__ typename Epi::Params ep) {
  using L = GemmSmem<BN, EpiSmem<Epi>::value>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty_bar = full_bar + L::kStages;
  uint64_t* tfull_bar = empty_bar + L::kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* prefix = reinterpret_cast<int*>(tmem_slot + 4);

  const int warp = ptx::warp_id();
  const int lane = ptx::lane_id();

  // tile prefix over groups
  const int G = p.num_groups;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int g = 0; g < G; ++g) {
      prefix[g] = acc;
      acc += group_tiles<kMode, BN>(p, g);
    }
    prefix[G] = acc;
  }
  if (warp == 4 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < L::kStages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 5) ptx::tmem_alloc<L::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = prefix[G];

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (ptx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        TileInfo ti;
        decode_tile<kMode, BN>(p, prefix, t, ti);
        if constexpr (kMode == kModeSwap && A_MN) { ti.ax = ti.m0; ti.ay = ti.g * p.Kw; }
        const int nkb = ceil_div(ti.k_len, kBK);
        for (int kb = 0; kb < nkb; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          ptx::mbar_arrive_expect_tx(&full_bar[stage], L::kStageBytes);
          if constexpr (A_MN) {
            ptx::tma_load_2d(sa, &tmA, &full_bar[stage], ti.ax, ti.ay + kb * kBK);
            ptx::tma_load_2d(sa + 8192, &tmA, &full_bar[stage], ti.ax + 64, ti.ay + kb * kBK);
          } else {
            ptx::tma_load_2d(sa, &tmA, &full_bar[stage], ti.ax + kb * kBK, ti.ay);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              ptx::tma_load_2d(sb + j * 8192, &tmB, &full_bar[stage], ti.bx + 64 * j, ti.by + kb * kBK);
          } else {
            ptx::tma_load_2d(sb, &tmB, &full_bar[stage], ti.bx + kb * kBK, ti.by);
          }
          if (++stage == L::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
      TileInfo ti;
      decode_tile<kMode, BN>(p, prefix, t, ti);
      const int buf = it & 1;
      const uint32_t use = static_cast<uint32_t>(it >> 1);
      ptx::mbar_wait(&tempty_bar[buf], (use & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + buf * BN;
      const uint32_t idesc = ptx::idesc_bf16(kBM, ti.n, A_MN, B_MN);
      const int nkb = ceil_div(ti.k_len, kBK);
      for (int kb = 0; kb < nkb; ++kb) {
        ptx::mbar_wait(&full_bar[stage], phase);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t sa = ptx::smem_u32(smem + stage * L::kStageBytes);
          const uint32_t sb = sa + L::kABytes;
          const int nk = min(kBK, ti.k_len - kb * kBK) / 16;
          for (int kk = 0; kk < nk; ++kk) {
            const uint64_t adesc = A_MN ? ptx::smem_desc_sw128(sa + kk * 2048, 8192, 1024)
                                        : ptx::smem_desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t bdesc = B_MN ? ptx::smem_desc_sw128(sb + kk * 2048, 8192, 1024)
                                        : ptx::smem_desc_sw128(sb + kk * 32, 16, 1024);
            ptx::mma_bf16(d_tmem, adesc, bdesc, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          ptx::mma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == L::kStages) { stage = 0; phase ^= 1; }
      }
      if (ptx::elect_one()) {
        if (nkb > 0) ptx::mma_commit(&tfull_bar[buf]);
        else ptx::mbar_arrive(&tfull_bar[buf]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue warps 0..3
    int it = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
      TileInfo ti;
      decode_tile<kMode, BN>(p, prefix, t, ti);
      const int buf = it & 1;
      const uint32_t use = static_cast<uint32_t>(it >> 1);
      ptx::mbar_wait(&tfull_bar[buf], use & 1);
      ptx::tc_fence_after();
      const uint32_t tmem_tile = tmem_base + buf * BN + (static_cast<uint32_t>(warp * 32) << 16);
      Epi::run(ep, p, ti, tmem_tile, warp, lane, smem + L::kEpiOffset);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty_bar[buf]);
    }
    Epi::finish(ep, warp, lane);
  }
  __syncthreads();
  if (warp == 5) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<L::kTmemCols>(tmem_base);
  }
}

// Convenience: 32 fp32 accumulator columns [c0, c0+32) of this thread's row.
__device__ __forceinline__ void load_acc32(uint32_t tmem_tile, int c0, float (&v)[32]) {
  uint32_t r[32];
  ptx::tmem_ld_32x32b_x32(tmem_tile + c0, r);
  ptx::tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace tamoe
