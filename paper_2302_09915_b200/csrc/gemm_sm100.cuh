// Persistent, warp-specialised tcgen05 GEMM engine shared by every dense
// contraction on the TA-MoE hot path (fused gate logits, expert FFN forward /
// dgrad / wgrad, gate dW and dX).
//
//   warps 0-7 : epilogue (warp w owns TMEM lanes 32(w%4).. and column half w/4)
//   warp 8    : TMA producer (one elected lane)
//   warp 9    : TMEM allocator + MMA issuer (one elected lane)
//
// A tile is always M=128 (TMEM lanes) x N<=BN (TMEM columns) x K (multiple of
// 16).  Operands are staged by TMA with 128-byte swizzle; each operand can be
// K-major (rows of 64 K-elements) or MN-major (64-element MN chunks of 64
// K-rows).  The fp32 accumulator is double buffered in TMEM so the epilogue of
// tile i overlaps the MMAs of tile i+1.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <type_traits>

#include "ptx.cuh"

namespace tamoe {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kEpiWarps = 8;
constexpr int kProducerWarp = kEpiWarps;
constexpr int kMmaWarp = kEpiWarps + 1;
constexpr int kGemmThreads = (kEpiWarps + 2) * 32;
constexpr int kMaxGroups = 256;  // groups (experts, or expert x source segments) per grouped launch

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
  int w_mod;             // kModeSwap: weight of group g is g % w_mod (0: g) -- (source, expert) segments
  int nsub;              // kModeWgrad: K of group g = sub-segments s*num_groups + g, s < nsub
  // kModeSwap chain: a second swap GEMM (Mw2 x Kw2, tensor maps / epilogue from EpiChain) whose token operand is
  // the first one's output, in the same persistent launch.  Its tiles follow the first GEMM's in the schedule; a
  // CTA reaching a second-GEMM tile waits until every first-GEMM tile of that (group, token tile) has stored its
  // rows (ready[g * ready_stride + tile] == ready_target), so CTAs that finish the first GEMM early start the
  // second one instead of idling at a kernel boundary.
  int chain;
  int Mw2, Kw2;
  int* ready;
  int ready_stride, ready_target;
};

// i-th tile of persistent cluster c out of nc (>= the tile count: done): round robin.  (A size-ordered,
// boustrophedon schedule and a split of the last round were measured slower / no faster: DESIGN.md 3.1.)
__device__ __forceinline__ int sched_tile(int i, int c, int nc) { return i * nc + c; }

struct TileInfo {
  int phase;   // kModeSwap chain: 0 first GEMM, 1 second
  int tj;      // kModeSwap: token tile index within the group
  int g;       // group
  int wg;      // weight index (kModeSwap)
  int m0, n0;  // offsets within the group's output
  int n;       // valid N columns (multiple of 16, <= BN)
  int k_len;   // K extent (multiple of 16)
  int ks;      // split index (kModeGateDw)
  int ax, ay;  // A TMA base coordinates (see load_stage)
  int bx, by;  // B TMA base coordinates
};

// Epilogues may declare `static constexpr int kWarpBytes` of scratch shared memory per epilogue warp.
// Epilogues that declare `static constexpr bool kEarlyRelease = true` free the TMEM accumulator
// themselves (right after copying it to registers) through the `release` callback.
template <class Epi, class = void>
struct EpiEarly {
  static constexpr bool value = false;
};
template <class Epi>
struct EpiEarly<Epi, decltype(void(Epi::kEarlyRelease))> {
  static constexpr bool value = Epi::kEarlyRelease;
};

// Epilogues that declare `static constexpr int kBufBytes` get two staging buffers per warp and are driven one
// tile ahead: Epi::prefetch(..., buffer) for tile i+1 is issued before the accumulator wait of tile i, so its
// loads are in flight during that tile's epilogue (Epi::prefetch_none() keeps async-group counts uniform).
template <class Epi, class = void>
struct EpiAhead {
  static constexpr bool value = false;
};
template <class Epi>
struct EpiAhead<Epi, decltype(void(Epi::kBufBytes))> {
  static constexpr bool value = true;
};

template <class Epi, class = void>
struct EpiSmem {
  static constexpr int warp = 0;
  static constexpr int value = 0;
};
template <class Epi>
struct EpiSmem<Epi, decltype(void(Epi::kWarpBytes))> {
  static constexpr int warp = Epi::kWarpBytes;
  static constexpr int value = Epi::kWarpBytes * kEpiWarps;
};

// Epilogues of a chained swap launch (EpiChain, expert.cu) declare `static constexpr bool kChained = true` and carry
// the second GEMM's tensor maps (tmA2 / tmB2) in their Params.
template <class Epi, class = void>
struct EpiChained {
  static constexpr bool value = false;
};
template <class Epi>
struct EpiChained<Epi, decltype(void(Epi::kChained))> {
  static constexpr bool value = Epi::kChained;
};

template <int BN, int kEpiBytes = 0, int kCG = 1>
struct GemmSmem {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = (BN / (kCG == 1 ? 1 : 2)) * kBK * 2;  // a CTA pair splits B's N between its CTAs
  static constexpr int kStageBytes = kABytes + kBBytes;
  // barriers: full[S], empty[S], tfull[2], tempty[2]; tmem addr; tile prefix; group starts / rows
  // barriers + TMEM address + the tile prefix; the group table itself is read from global memory (L1-resident),
  // so the pipeline gets every byte it can (one more stage for the FFN forward / wgrad / K = 4096 GEMMs)
  static constexpr int kMiscBytes = (2 * 8 + 4) * 8 + 16 + (kMaxGroups + 1) * 4;
  static constexpr int kBudget = 227 * 1024 - ((kEpiBytes + 1023) / 1024) * 1024 - kMiscBytes - 1024;
#ifdef TAMOE_MAX_STAGES
  static constexpr int kMaxStages = TAMOE_MAX_STAGES;  // A/B experiments only
#else
  static constexpr int kMaxStages = 8;
#endif
  static constexpr int kStages = (kBudget / kStageBytes < kMaxStages) ? kBudget / kStageBytes : kMaxStages;
  static_assert(kStages >= 2, "not enough shared memory for the pipeline");
  static constexpr int kEpiOffset = kStages * kStageBytes;
  static constexpr int kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr int kBarOffset = kEpiOffset + ((kEpiBytes + 1023) / 1024) * 1024;
  static constexpr int kTotal = kBarOffset + kMiscBytes + 1024;  // + alignment slack
  static_assert(kTotal <= 227 * 1024, "shared memory over the sm_100 per-CTA limit");
};

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Token tiles of a swap-mode group: rows split into ceil(rows / BN) balanced tiles (multiples of 16).
template <int BN>
__device__ __forceinline__ int swap_ntiles(int rows) { return ceil_div(rows, BN); }
template <int BN>
__device__ __forceinline__ int swap_nsize(int rows) {
  const int nb = ceil_div(rows, BN);
  return nb > 0 ? ((ceil_div(rows, nb) + 15) & ~15) : 0;
}

// Number of tiles of group g (device side; prefix built once per CTA).  `rows` = seg_rows[g].
template <int kMode, int BN, int kCG = 1>
__device__ __forceinline__ int group_tiles(const GemmParams& p, int rows) {
  if constexpr (kMode == kModeSwap) {
    return swap_ntiles<BN>(rows);  // token tiles; a tile = (m block, token tile), see decode_tile
  } else if constexpr (kMode == kModeWgrad) {
    return (p.Mw / (kBM * kCG)) * (p.Nw / BN);
  } else if constexpr (kMode == kModeGate) {
    return p.procs * ceil_div(p.tokens_per_proc, kBM);
  } else if constexpr (kMode == kModeGateDw) {
    return p.procs * (p.Mw / kBM) * (p.Nw / BN) * p.k_split;
  } else {
    return p.procs * ceil_div(p.tokens_per_proc, kBM) * (p.Nw / BN);
  }
}

// Tiles of a swap launch: every group's (m block, token tile) pairs, m-block-major within the group; with a chain,
// the second GEMM's tiles follow all of the first's.  prefix[] holds the groups' token-tile prefix.
template <int BN, int kCG>
__device__ __forceinline__ int swap_total_tiles(const GemmParams& p, const int* prefix) {
  const int nt = prefix[p.num_groups];
  return (p.Mw / (kBM * kCG)) * nt + (p.chain ? (p.Mw2 / (kBM * kCG)) * nt : 0);
}

template <int kMode, int BN, int kCG = 1>
__device__ __forceinline__ void decode_tile(const GemmParams& p, const int* prefix, const int* s_start,
                                            const int* s_rows, int t, TileInfo& ti) {
  ti.phase = 0;
  ti.tj = 0;
  if constexpr (kMode == kModeSwap) {
    int MB = p.Mw / (kBM * kCG), Mw = p.Mw, Kw = p.Kw;
    const int t1 = MB * prefix[p.num_groups];
    if (p.chain && t >= t1) {
      t -= t1;
      ti.phase = 1;
      MB = p.Mw2 / (kBM * kCG);
      Mw = p.Mw2;
      Kw = p.Kw2;
    }
    int lo = 0, hi = p.num_groups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (MB * prefix[mid] <= t) lo = mid; else hi = mid - 1;
    }
    const int g = lo;
    const int r = t - MB * prefix[g];
    const int rows = s_rows[g];
    const int nb = swap_ntiles<BN>(rows);
    const int ns = swap_nsize<BN>(rows);
    const int mb = r / nb, nbk = r % nb;
    ti.g = g;
    ti.ks = 0;
    ti.tj = nbk;
    ti.wg = p.w_mod > 0 ? g % p.w_mod : g;
    ti.m0 = mb * kBM * kCG;
    ti.n0 = nbk * ns;
    ti.n = min(ns, rows - ti.n0);
    ti.k_len = Kw;
    // A (weights): K-major -> (k, g*Mw + m0) ; MN-major -> (m0, g*Kw + k) (the producer localises per CTA)
    ti.ax = 0; ti.ay = g * Mw + ti.m0;
    ti.bx = 0; ti.by = s_start[g] + ti.n0;
    return;
  }
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
  if constexpr (kMode == kModeWgrad) {
    const int nb = p.Nw / BN;
    ti.m0 = (r / nb) * kBM * kCG;
    ti.n0 = (r % nb) * BN;
    ti.n = BN;
    ti.k_len = 0;
    for (int sub = 0; sub < p.nsub; ++sub) ti.k_len += s_rows[sub * p.num_groups + g];
    ti.ax = ti.m0; ti.ay = s_start[g];
    ti.bx = ti.n0; ti.by = s_start[g];
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
//                const TileInfo&, uint32_t tmem_tile /*lane 32q, col 0 of this tile*/, int q /*lane quarter*/,
//                int h /*column half*/, int lane, uint8_t* smem /*this warp's kWarpBytes*/, const int* s_start);
//                static __device__ void prefetch(...same without tmem_tile...);   // before the accumulator wait
//                static __device__ void finish(const Params&, int lane); };
template <int kMode, int BN, bool A_MN, bool B_MN, class Epi, int kCG>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const GemmParams p, const __grid_constant__ typename Epi::Params ep) {
  static_assert(kCG == 1 || kMode == kModeSwap || kMode == kModeWgrad, "CTA pairs only for grouped modes");
  // kCG = 4: two CTA pairs per cluster on adjacent weight blocks of the same token tile; the token (B) operand
  // is loaded once per cluster and multicast to both pairs (halves its L2 -> SMEM traffic)
  static_assert(kCG != 4 || (kMode == kModeSwap && !B_MN), "pair multicast only for K-major swap GEMMs");
  static_assert(kCG == 1 || kCG == 2 || kCG == 4, "cluster of 1 CTA, one pair or two pairs");
  constexpr int kCGm = kCG == 1 ? 1 : 2;  // CTAs per tcgen05.mma (cta_group)
  using L = GemmSmem<BN, EpiSmem<Epi>::value, kCG>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty_bar = full_bar + L::kStages;
  uint64_t* tfull_bar = empty_bar + L::kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* prefix = reinterpret_cast<int*>(tmem_slot + 4);
  // group table: global (seg_start / seg_rows of the grouped modes; the gate modes have one implicit group)
  const int* s_start = p.seg_start;
  const int* s_rows = p.seg_rows;

  const int warp = ptx::warp_id();
  const int lane = ptx::lane_id();
  const uint32_t rank = kCG > 1 ? ptx::cluster_ctarank() : 0u;
  const uint32_t pair_base = rank & ~1u;  // rank of this CTA's pair leader
  const bool leader = (rank & 1u) == 0;
  const int cluster_id = blockIdx.x / kCG;
  const int num_clusters = gridDim.x / kCG;

  // programmatic dependent launch: let the next kernel of the step get scheduled as SMs free up, and set up
  // barriers / TMEM / tensor maps (no dependent data) before waiting for the previous kernel's results
  ptx::pdl_trigger();
  if (warp == kProducerWarp && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < L::kStages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], kCG == 4 ? 2 : 1);  // kCG 4: both pairs read every stage
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], kEpiWarps * kCGm);
    }
    ptx::fence_barrier_init();
  }
  if (warp == kMmaWarp) {
    if constexpr (kCG > 1) ptx::tmem_alloc_cg2<L::kTmemCols>(tmem_slot);
    else ptx::tmem_alloc<L::kTmemCols>(tmem_slot);
  }
  ptx::pdl_wait();
  // warp-parallel prefix of the groups' tile counts (smem)
  const int G = p.num_groups;
  constexpr bool grouped = (kMode == kModeSwap || kMode == kModeWgrad);
  if (warp == 0) {
    int carry = 0;
    for (int g0 = 0; g0 < G; g0 += 32) {
      const int g = g0 + lane;
      const int c = g < G ? group_tiles<kMode, BN, kCG>(p, grouped ? s_rows[g] : 0) : 0;
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (g < G) prefix[g] = carry + x - c;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) prefix[G] = carry;
  }
  ptx::tc_fence_before();
  if constexpr (kCG > 1) ptx::cluster_sync();
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = kMode == kModeSwap ? swap_total_tiles<BN, kCG>(p, prefix) : prefix[G];

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ TMA producer (both CTAs of a pair)
    if (ptx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      // this CTA's operand coordinates of a decoded tile
      auto localize = [&](TileInfo& ti) {
        const int my_m0 = ti.m0 + static_cast<int>(rank) * kBM;
        if constexpr (kMode == kModeSwap) {
          const int Mw = ti.phase ? p.Mw2 : p.Mw, Kw = ti.phase ? p.Kw2 : p.Kw;
          if constexpr (A_MN) { ti.ax = my_m0; ti.ay = ti.wg * Kw; }
          else { ti.ay = ti.wg * Mw + my_m0; }
          ti.by += static_cast<int>(rank & 1u) * (ti.n / kCGm);  // this CTA's half of the token tile
        } else if constexpr (kMode == kModeWgrad) {
          ti.ax = my_m0;
          ti.bx += static_cast<int>(rank) * (BN / kCG);
        }
      };
      for (int i = 0;; ++i) {
        const int t = sched_tile(i, cluster_id, num_clusters);
        if (t >= total_tiles) break;
        TileInfo ti;
        decode_tile<kMode, BN, kCG>(p, prefix, s_start, s_rows, t, ti);
        localize(ti);
        const CUtensorMap* mA = &tmA;
        const CUtensorMap* mB = &tmB;
        if constexpr (EpiChained<Epi>::value) {
          if (ti.phase) {
            mA = &ep.tmA2;
            mB = &ep.tmB2;
            // the second GEMM's token operand is the first's output: every first-GEMM tile of this (group, token
            // tile) must have stored its rows
            ptx::wait_counter_geq(p.ready + ti.g * p.ready_stride + ti.tj, p.ready_target);
          }
        }
        // K ranges: wgrad walks the group's (source) sub-segments; every other mode has one range
        const int nsub = (kMode == kModeWgrad) ? p.nsub : 1;
        for (int sub = 0; sub < nsub; ++sub) {
          int klen = ti.k_len, krow = 0;
          if constexpr (kMode == kModeWgrad) {
            klen = s_rows[sub * G + ti.g];
            krow = s_start[sub * G + ti.g];
            ti.ay = krow;
            ti.by = krow;
          }
          const int nkb = ceil_div(klen, kBK);
          for (int kb = 0; kb < nkb; ++kb) {
            ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sa = smem + stage * L::kStageBytes;
            uint8_t* sb = sa + L::kABytes;
            if (leader) ptx::mbar_arrive_expect_tx(&full_bar[stage], kCGm * L::kStageBytes);
            if constexpr (kCG > 1) {
              const uint32_t bar = ptx::mapa(&full_bar[stage], pair_base);
              if constexpr (A_MN) {
                ptx::tma_load_2d_cg2(sa, mA, bar, ti.ax, ti.ay + kb * kBK);
                ptx::tma_load_2d_cg2(sa + 8192, mA, bar, ti.ax + 64, ti.ay + kb * kBK);
              } else {
                ptx::tma_load_2d_cg2(sa, mA, bar, ti.ax + kb * kBK, ti.ay);
              }
              if constexpr (kCG == 4) {
                // this pair loads one half of the CTA-half token box; both pairs' CTAs of the same half get it
                const int pp = static_cast<int>(rank >> 1);
                const uint16_t mask = static_cast<uint16_t>((1u << (rank & 1u)) | (1u << ((rank & 1u) + 2)));
                ptx::tma_load_2d_cg2_mc(sb + pp * (L::kBBytes / 2), mB, bar, ti.bx + kb * kBK,
                                        ti.by + pp * (BN / 4), mask);
              } else if constexpr (B_MN) {
#pragma unroll
                for (int j = 0; j < BN / 128; ++j)
                  ptx::tma_load_2d_cg2(sb + j * 8192, mB, bar, ti.bx + 64 * j, ti.by + kb * kBK);
              } else {
                ptx::tma_load_2d_cg2(sb, mB, bar, ti.bx + kb * kBK, ti.by);
              }
            } else {
              if constexpr (A_MN) {
                ptx::tma_load_2d(sa, mA, &full_bar[stage], ti.ax, ti.ay + kb * kBK);
                ptx::tma_load_2d(sa + 8192, mA, &full_bar[stage], ti.ax + 64, ti.ay + kb * kBK);
              } else {
                ptx::tma_load_2d(sa, mA, &full_bar[stage], ti.ax + kb * kBK, ti.ay);
              }
              if constexpr (B_MN) {
#pragma unroll
                for (int j = 0; j < BN / 64; ++j)
                  ptx::tma_load_2d(sb + j * 8192, mB, &full_bar[stage], ti.bx + 64 * j, ti.by + kb * kBK);
              } else {
                ptx::tma_load_2d(sb, mB, &full_bar[stage], ti.bx + kb * kBK, ti.by);
              }
            }
            if (++stage == L::kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (pair leader only)
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (;; ++it) {
        const int t = sched_tile(it, cluster_id, num_clusters);
        if (t >= total_tiles) break;
        TileInfo ti;
        decode_tile<kMode, BN, kCG>(p, prefix, s_start, s_rows, t, ti);
        const int buf = it & 1;
        const uint32_t use = static_cast<uint32_t>(it >> 1);
        ptx::mbar_wait(&tempty_bar[buf], (use & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        const uint32_t idesc = ptx::idesc_bf16(kBM * kCGm, ti.n, A_MN, B_MN);
        const int nsub = (kMode == kModeWgrad) ? p.nsub : 1;
        uint32_t acc = 0;
        int nkb_total = 0;
        for (int sub = 0; sub < nsub; ++sub) {
          const int klen = (kMode == kModeWgrad) ? s_rows[sub * G + ti.g] : ti.k_len;
          const int nkb = ceil_div(klen, kBK);
          nkb_total += nkb;
          for (int kb = 0; kb < nkb; ++kb) {
            ptx::mbar_wait(&full_bar[stage], phase);
            ptx::tc_fence_after();
            const int nk = min(kBK, klen - kb * kBK) / 16;  // warp-uniform
            if (ptx::elect_one()) {
              const uint32_t sa = ptx::smem_u32(smem + stage * L::kStageBytes);
              const uint32_t sb = sa + L::kABytes;
              for (int kk = 0; kk < nk; ++kk) {
                const uint64_t adesc = A_MN ? ptx::smem_desc_sw128(sa + kk * 2048, 8192, 1024)
                                            : ptx::smem_desc_sw128(sa + kk * 32, 16, 1024);
                const uint64_t bdesc = B_MN ? ptx::smem_desc_sw128(sb + kk * 2048, 8192, 1024)
                                            : ptx::smem_desc_sw128(sb + kk * 32, 16, 1024);
                const uint32_t accum = (acc | static_cast<uint32_t>(kk > 0)) ? 1u : 0u;
                if constexpr (kCG > 1) ptx::mma_bf16_cg2(d_tmem, adesc, bdesc, idesc, accum);
                else ptx::mma_bf16(d_tmem, adesc, bdesc, idesc, accum);
              }
              if constexpr (kCG == 4) ptx::mma_commit_cg2(&empty_bar[stage], 0xF);  // B came from both pairs
              else if constexpr (kCG == 2) ptx::mma_commit_cg2(&empty_bar[stage], 0x3);
              else ptx::mma_commit(&empty_bar[stage]);
            }
            if (nk > 0) acc = 1u;
            __syncwarp();
            if (++stage == L::kStages) { stage = 0; phase ^= 1; }
          }
        }
        const int nkb = nkb_total;
        if (ptx::elect_one()) {
          if (nkb > 0) {
            if constexpr (kCG > 1) ptx::mma_commit_cg2(&tfull_bar[buf], static_cast<uint16_t>(0x3u << pair_base));
            else ptx::mma_commit(&tfull_bar[buf]);
          } else {
            if constexpr (kCG > 1) {
              ptx::mbar_arrive_remote(ptx::mapa(&tfull_bar[buf], pair_base));
              ptx::mbar_arrive_remote(ptx::mapa(&tfull_bar[buf], pair_base + 1));
            } else {
              ptx::mbar_arrive(&tfull_bar[buf]);
            }
          }
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps 0..7 (both CTAs)
    const int q = warp & 3, h = warp >> 2;
    uint8_t* wsm = smem + L::kEpiOffset + warp * EpiSmem<Epi>::warp;
    int it = 0;
    if constexpr (EpiAhead<Epi>::value) {
      static_assert(!EpiEarly<Epi>::value, "tile-ahead epilogues release TMEM after run()");
      TileInfo nx;
      if (sched_tile(0, cluster_id, num_clusters) < total_tiles) {
        decode_tile<kMode, BN, kCG>(p, prefix, s_start, s_rows, sched_tile(0, cluster_id, num_clusters),
                                    nx);
        nx.m0 += static_cast<int>(rank) * kBM;
        Epi::prefetch(ep, p, nx, q, h, lane, wsm, s_start);
      }
      for (;; ++it) {
        if (sched_tile(it, cluster_id, num_clusters) >= total_tiles) break;
        const TileInfo ti = nx;
        const int tn = sched_tile(it + 1, cluster_id, num_clusters);
        if (tn < total_tiles) {
          decode_tile<kMode, BN, kCG>(p, prefix, s_start, s_rows, tn, nx);
          nx.m0 += static_cast<int>(rank) * kBM;
          Epi::prefetch(ep, p, nx, q, h, lane, wsm + ((it + 1) & 1) * Epi::kBufBytes, s_start);
        } else {
          Epi::prefetch_none();
        }
        const int buf = it & 1;
        const uint32_t use = static_cast<uint32_t>(it >> 1);
        ptx::mbar_wait(&tfull_bar[buf], use & 1);
        ptx::tc_fence_after();
        const uint32_t tmem_tile = tmem_base + buf * BN + (static_cast<uint32_t>(q * 32) << 16);
        Epi::run(ep, p, ti, tmem_tile, q, h, lane, wsm + (it & 1) * Epi::kBufBytes, s_start);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kCG > 1) ptx::mbar_arrive_remote(ptx::mapa(&tempty_bar[buf], pair_base));
          else ptx::mbar_arrive(&tempty_bar[buf]);
        }
      }
    } else if constexpr (EpiChained<Epi>::value) {
      // chained launch: the first GEMM's tiles (epilogue Epi::First), then the second's (Epi::Second) -- two loops,
      // each inlining one epilogue body
      auto phase_loop = [&](auto ph) {
        constexpr int PH = decltype(ph)::value;
        using E = typename std::conditional<PH == 0, typename Epi::First, typename Epi::Second>::type;
        const auto& epp = Epi::params(ep, ph);
        for (;; ++it) {
          const int t = sched_tile(it, cluster_id, num_clusters);
          if (t >= total_tiles) break;
          TileInfo ti;
          decode_tile<kMode, BN, kCG>(p, prefix, s_start, s_rows, t, ti);
          if (ti.phase != PH) break;  // (first loop) this CTA's second-GEMM tiles start here
          ti.m0 += static_cast<int>(rank) * kBM;
          const int buf = it & 1;
          const uint32_t use = static_cast<uint32_t>(it >> 1);
          E::prefetch(epp, p, ti, q, h, lane, wsm, s_start);
          ptx::mbar_wait(&tfull_bar[buf], use & 1);
          ptx::tc_fence_after();
          const uint32_t tmem_tile = tmem_base + buf * BN + (static_cast<uint32_t>(q * 32) << 16);
          auto release = [&]() {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if constexpr (kCG > 1) ptx::mbar_arrive_remote(ptx::mapa(&tempty_bar[buf], pair_base));
              else ptx::mbar_arrive(&tempty_bar[buf]);
            }
          };
          E::run(epp, p, ti, tmem_tile, q, h, lane, wsm, s_start, release);
          if constexpr (PH == 0) {
            // this warp's rows of a first-GEMM tile are in global memory: count them for the second GEMM's producers
            if (lane == 0) {
              ptx::bulk_wait<0>();
              ptx::fence_proxy_async_global();
              __threadfence();
              atomicAdd(p.ready + ti.g * p.ready_stride + ti.tj, 1);
            }
            __syncwarp();
          }
        }
      };
      phase_loop(std::integral_constant<int, 0>{});
      phase_loop(std::integral_constant<int, 1>{});
      Epi::First::finish(ep.p0, lane);
      Epi::Second::finish(ep.p1, lane);
    } else {
    for (;; ++it) {
      const int t = sched_tile(it, cluster_id, num_clusters);
      if (t >= total_tiles) break;
      TileInfo ti;
      decode_tile<kMode, BN, kCG>(p, prefix, s_start, s_rows, t, ti);
      ti.m0 += static_cast<int>(rank) * kBM;  // this CTA's 128 accumulator rows
      const int buf = it & 1;
      const uint32_t use = static_cast<uint32_t>(it >> 1);
      Epi::prefetch(ep, p, ti, q, h, lane, wsm, s_start);
      ptx::mbar_wait(&tfull_bar[buf], use & 1);
      ptx::tc_fence_after();
      const uint32_t tmem_tile = tmem_base + buf * BN + (static_cast<uint32_t>(q * 32) << 16);
      auto release = [&]() {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kCG > 1) ptx::mbar_arrive_remote(ptx::mapa(&tempty_bar[buf], pair_base));
          else ptx::mbar_arrive(&tempty_bar[buf]);
        }
      };
      if constexpr (EpiEarly<Epi>::value) {
        Epi::run(ep, p, ti, tmem_tile, q, h, lane, wsm, s_start, release);
      } else {
        Epi::run(ep, p, ti, tmem_tile, q, h, lane, wsm, s_start);
        release();
      }
    }
    Epi::finish(ep, lane);
    }
  }
  if constexpr (kCG > 1) ptx::cluster_sync();
  else __syncthreads();
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    if constexpr (kCG > 1) ptx::tmem_dealloc_cg2<L::kTmemCols>(tmem_base);
    else ptx::tmem_dealloc<L::kTmemCols>(tmem_base);
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
