// Expert histogram / scan / capacity / permute kernels.
//
// Replaces the counting and capacity parts of topk_route (gate.cpp:138-199)
// and the token movement the reference leaves implicit.  Bucket order inside
// an expert is ascending (process, token, slot) -- the reference's bucket
// insertion order (gate.cpp:160-164, 181-185) -- and capacity keeps the best
// (score desc, process asc, token asc) picks (gate.cpp:140-149) via an exact
// radix select on the fp64 score bits, so kept sets are bit-identical.
#include <cuda_bf16.h>

#include <climits>
#include <cstdint>

#include "common.hpp"
#include "ptx.cuh"
#include "route.hpp"

namespace tamoe {

namespace {

// In-place exclusive scan of smem a[0..n); returns the total.  All threads of the block must call.
__device__ int block_excl_scan(int* a, int n, int* wtmp) {
  const int nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int b = threadIdx.x * per;
  const int e = min(n, b + per);
  int local = 0;
  for (int i = b; i < e; ++i) local += a[i];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (nt + 31) >> 5;
  int x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wtmp[w] = x;
  __syncthreads();
  if (w == 0) {
    int v = lane < nw ? wtmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane < nw) wtmp[lane] = v;
  }
  __syncthreads();
  int base = (w > 0 ? wtmp[w - 1] : 0) + x - local;
  for (int i = b; i < e; ++i) {
    const int t = a[i];
    a[i] = base;
    base += t;
  }
  const int total = wtmp[nw - 1];
  __syncthreads();
  return total;
}

// Mean probabilities of expert e for every process (gate.cpp:115): the 32-token group sums msum4 added in a
// fixed block-parallel order, / S.  All threads of the block must call.
__device__ void mean_probs_column(const RouteDims& d, const RouteBuffers& b, int e) {
  __shared__ double dred[32];
  const int N = d.N;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int pr = 0; pr < d.P; ++pr) {
    double m = 0.0;
    const int t0 = pr * d.TB * 4, t1 = (pr + 1) * d.TB * 4;
    for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) m += b.msum4[static_cast<long long>(t) * N + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    if (lane == 0) dred[w] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      double mt = 0.0;
      for (int i = 0; i < nw; ++i) mt += dred[i];
      b.mean_probs[pr * N + e] = mt / d.S;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- scan
// One CTA per expert: exclusive prefix of the per-(tile, warp) pick counts in
// (process, token) order -> base4, plus per-(process, expert) bucket ranges.
constexpr int kScanThreads = 512;

__global__ void __launch_bounds__(kScanThreads) route_scan_kernel(RouteDims d, RouteBuffers b, int direct) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ int wsum[32];
  __shared__ int carry_s;
  const int e = blockIdx.x, N = d.N;
  const int entries = d.tiles() * 4;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int j0 = 0; j0 < entries; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    const int c = j < entries ? b.hist4[static_cast<long long>(j) * N + e] : 0;
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int before = carry_s;
    for (int i = 0; i < w; ++i) before += wsum[i];
    const int excl = before + x - c;
    if (j < entries) {
      b.base4[static_cast<long long>(j) * N + e] = excl;
      if (j % (d.TB * 4) == 0) b.bucket_start[(j / (d.TB * 4)) * N + e] = excl;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < nw; ++i) carry_s += wsum[i];
    __syncthreads();
  }
  if (threadIdx.x == 0) b.list_count[e] = carry_s;
  __syncthreads();
  for (int pr = threadIdx.x; pr < d.P; pr += blockDim.x) {
    const int st = b.bucket_start[pr * N + e];
    const int en = pr + 1 < d.P ? b.bucket_start[(pr + 1) * N + e] : carry_s;
    b.bucket_count[pr * N + e] = en - st;
    if (direct) {  // no capacity: every pick is kept
      b.counts[pr * N + e] = en - st;
      b.dropped[pr * N + e] = 0;
    }
  }
  if (direct) mean_probs_column(d, b, e);
}

// ---------------------------------------------------------------- bucket
// One CTA per 128-token tile.  Position of a pick in its expert's list =
// list_start[e] + picks to e in earlier (tile, warp) slots + earlier lanes of its warp.
__global__ void __launch_bounds__(kRouteTile) route_bucket_kernel(RouteDims d, RouteBuffers b, int direct) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  extern __shared__ int sm[];
  const int N = d.N, k = d.k;
  int* wbase = sm;                     // [4*N]
  int* sel = wbase + 4 * N;            // [128*k]
  int* wtmp = sel + kRouteTile * k;    // [32]
  int* ls = wtmp + 32;                 // [N]
  const int tile = blockIdx.x;
  for (int e = threadIdx.x; e < N; e += blockDim.x) ls[e] = b.list_count[e];
  __syncthreads();
  block_excl_scan(ls, N, wtmp);
  for (int i = threadIdx.x; i < 4 * N; i += blockDim.x) {
    const int w = i / N, e = i % N;
    wbase[i] = ls[e] + b.base4[(static_cast<long long>(tile) * 4 + w) * N + e];
  }
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < N; e += blockDim.x) b.list_start[e] = ls[e];
  const int proc = tile / d.TB;
  const int tok = (tile % d.TB) * kRouteTile + threadIdx.x;
  const bool valid = tok < d.S;
  const long long gtok = static_cast<long long>(proc) * d.S + tok;
  for (int j = 0; j < k; ++j) sel[threadIdx.x * k + j] = valid ? b.idx[gtok * k + j] : -1;
  __syncthreads();
  if (!valid) return;
  const int w = threadIdx.x >> 5;
  for (int a = 0; a < k; ++a) {
    const int e = sel[threadIdx.x * k + a];
    int r = 0;
    for (int l = w * 32; l < threadIdx.x; ++l)
      for (int j = 0; j < k; ++j) r += (sel[l * k + j] == e);
    const int pos = wbase[w * N + e] + r;
    const int pick = static_cast<int>(gtok * k + a);
    if (direct) {  // no capacity: the bucket lists are the compacted kept lists
      b.clist[pos] = pick;
      b.kept[pick] = 1;
    } else {
      b.list_pick[pos] = pick;
      b.list_score[pos] = b.score[pick];
    }
  }
}

// ---------------------------------------------------------------- capacity
// One CTA per expert.  For every capacity domain (bucket) over budget, an exact
// 8-pass radix select on the fp64 score bits finds the cap-th best score v;
// keep score > v, plus the first (cap - #greater) picks with score == v in list
// order (= process asc, token asc).
constexpr int kCapThreads = 512;

__device__ __forceinline__ unsigned long long score_key(double s) {
  // scores are probabilities >= 0: the IEEE bits are monotone
  return static_cast<unsigned long long>(__double_as_longlong(s));
}

__global__ void __launch_bounds__(kCapThreads) route_capacity_kernel(RouteDims d, RouteBuffers b, int mode,
                                                                     const int* __restrict__ caps) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ int hist[256];
  __shared__ int wtmp[32];
  __shared__ int sh_digit, sh_need;
  __shared__ int carry;
  const int e = blockIdx.x;
  const int N = d.N;
  const int ls = b.list_start[e];
  const int nb = mode == 1 ? 1 : (mode == 4 ? 0 : d.P);
  if (mode == 4)  // external decision (expert-parallel global capacity): b.kept holds the flags per pick
    for (int j = threadIdx.x; j < b.list_count[e]; j += blockDim.x) b.list_keep[ls + j] = b.kept[b.list_pick[ls + j]];
  // pass A: per bucket select + keep flags
  for (int bk = 0; bk < nb; ++bk) {
    const int bs = mode == 1 ? 0 : b.bucket_start[bk * N + e];
    const int bc = mode == 1 ? b.list_count[e] : b.bucket_count[bk * N + e];
    const int cap = mode == 0 ? INT_MAX : max(caps[bk * N + e], 0);
    const double* sc = b.list_score + ls + bs;
    uint8_t* keep = b.list_keep + ls + bs;
    if (bc <= cap) {
      for (int j = threadIdx.x; j < bc; j += blockDim.x) keep[j] = 1;
      continue;
    }
    unsigned long long prefix = 0, mask = 0;
    int need = cap;  // elements still to take from the top among the candidates
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (int j = threadIdx.x; j < bc; j += blockDim.x) {
        const unsigned long long key = score_key(sc[j]);
        if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int cum = 0, dg = 0;
        for (dg = 255; dg > 0; --dg) {
          if (cum + hist[dg] >= need) break;
          cum += hist[dg];
        }
        sh_digit = dg;
        sh_need = need - cum;
      }
      __syncthreads();
      prefix |= static_cast<unsigned long long>(sh_digit) << shift;
      mask |= 255ull << shift;
      need = sh_need;
      __syncthreads();
    }
    // need = how many picks with key == prefix to keep (in list order)
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int j0 = 0; j0 < bc; j0 += blockDim.x) {
      const int j = j0 + threadIdx.x;
      unsigned long long key = 0;
      int eq = 0;
      if (j < bc) {
        key = score_key(sc[j]);
        eq = key == prefix;
      }
      // exclusive rank of equality flags inside the block
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
      const unsigned bal = __ballot_sync(0xffffffffu, eq);
      const int in_warp = __popc(bal & ((1u << lane) - 1));
      if (lane == 0) wtmp[w] = __popc(bal);
      __syncthreads();
      int before = carry;
      for (int ww = 0; ww < w; ++ww) before += wtmp[ww];
      if (j < bc) keep[j] = (key > prefix) || (eq && (before + in_warp) < need);
      __syncthreads();
      if (threadIdx.x == 0) {
        int s = 0;
        for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) s += wtmp[ww];
        carry += s;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  // pass B: compaction over the whole expert list (stable), counts, kept / pos of drops
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int total = b.list_count[e];
  for (int j0 = 0; j0 < total; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    const int kp = j < total ? b.list_keep[ls + j] : 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, kp);
    if (lane == 0) wtmp[w] = __popc(bal);
    __syncthreads();
    int before = carry;
    for (int ww = 0; ww < w; ++ww) before += wtmp[ww];
    if (j < total) {
      const int pick = b.list_pick[ls + j];
      b.kept[pick] = static_cast<uint8_t>(kp);
      if (kp) b.clist[ls + before + __popc(bal & ((1u << lane) - 1))] = pick;
      else b.pos[pick] = -1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = 0;
      for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) s += wtmp[ww];
      carry += s;
    }
    __syncthreads();
  }
  // per-bucket kept / dropped counts (block-parallel) and mean probabilities (fixed-order sums)
  __shared__ int ired[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int pr = 0; pr < d.P; ++pr) {
    const int bs = b.bucket_start[pr * N + e], bc = b.bucket_count[pr * N + e];
    int kc = 0;
    if (mode == 1 || mode == 4) {
      for (int j = threadIdx.x; j < bc; j += blockDim.x) kc += b.list_keep[ls + bs + j];
    } else if (threadIdx.x == 0) {
      kc = mode == 0 ? bc : min(bc, max(caps[pr * N + e], 0));  // exactly cap picks survive
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kc += __shfl_xor_sync(0xffffffffu, kc, o);
    if (lane == 0) ired[w] = kc;
    __syncthreads();
    if (threadIdx.x == 0) {
      int kt = 0;
      for (int i = 0; i < nw; ++i) kt += ired[i];
      b.counts[pr * N + e] = kt;
      b.dropped[pr * N + e] = bc - kt;
    }
    __syncthreads();
  }
  mean_probs_column(d, b, e);
}

// ---------------------------------------------------------------- permute
// One warp per destination row of the padded expert-sorted buffer.
constexpr int kPermWarps = 8;

__global__ void __launch_bounds__(kPermWarps * 32) route_permute_kernel(RouteDims d, RouteBuffers b,
                                                                        const __nv_bfloat16* __restrict__ x, int dx,
                                                                        const __grid_constant__ PeerBufs xp, int r_max,
                                                                        const __grid_constant__ PeerBufs zrows,
                                                                        int has_z, int zdim, RowMap map,
                                                                        const __grid_constant__ PeerInts codes,
                                                                        int has_codes, int me, int trash_row) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  extern __shared__ int sm[];
  const int N = d.N;
  int* start = sm;          // [N]
  int* cnt = start + N;     // [N]
  int* wtmp = cnt + N;      // [32]
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    int c = 0;
    for (int pr = 0; pr < d.P; ++pr) c += b.counts[pr * N + e];
    cnt[e] = c;
    start[e] = (c + 15) & ~15;
  }
  __syncthreads();
  const int total = block_excl_scan(start, N, wtmp);
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
      b.seg_start[e] = start[e];
      b.seg_rows[e] = (cnt[e] + 15) & ~15;
    }
    if (threadIdx.x == 0) *b.total_rows = total;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows = min(total, r_max);
  // Under expert parallelism the rows are owner-major.  With at least one block per owner, the blocks are dealt
  // to the owners round robin (block b serves owner (me + b) % W), so this rank's stores to every peer and its local
  // copies run concurrently from the start and, rank by rank, the peers are offset (no incast); otherwise every rank
  // starts at its own owner segment and walks the owners cyclically.
  auto move_row = [&](int r) {
    int lo = 0, hi = N - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (start[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int e = lo;
    const int j = r - start[e];
    const int dst_rank = map.rank_of(e);
    const long long drow = map.P == 1 ? r : static_cast<long long>(r) - start[e] + map.dst_off[e];
    uint4* dst = reinterpret_cast<uint4*>(xp.p[dst_rank] + drow * dx);
    const int nv = dx / 8;
    const int rep = xp.rep[dst_rank];
    if (j < cnt[e]) {
      const int pick = b.clist[b.list_start[e] + j];
      const long long tok = pick / d.k;
      if (lane == 0) {
        b.pos[pick] = r;
        if (has_codes) codes.p[dst_rank][drow] = (me << kPushRowBits) | pick;
      }
      const uint4* src = reinterpret_cast<const uint4*>(x + tok * dx);
      // whole row in registers first (up to 8 x 16 B per lane), then the stores back to back
      constexpr int kU = 8;
      for (int v0 = lane; v0 < nv; v0 += 32 * kU) {
        uint4 t[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (v0 + 32 * u < nv) t[u] = __ldg(src + v0 + 32 * u);
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (v0 + 32 * u < nv) dst[v0 + 32 * u] = t[u];
        if (rep > 1) {
#pragma unroll
          for (int u = 0; u < kU; ++u)
            if (v0 + 32 * u < nv) store_repeat(dst + v0 + 32 * u, t[u], rep);
        }
      }
    } else {
      if (lane == 0 && has_codes) codes.p[dst_rank][drow] = (me << kPushRowBits) | trash_row;
      const uint4 z = make_uint4(0, 0, 0, 0);
      for (int v = lane; v < nv; v += 32) {
        dst[v] = z;
        if (rep > 1) store_repeat(dst + v, z, rep);
      }
      if (has_z) {
        uint4* zd = reinterpret_cast<uint4*>(zrows.p[dst_rank] + drow * zdim);
        for (int v = lane; v < zdim / 8; v += 32) zd[v] = z;
      }
    }
  };
  const int W = map.P;
  if (W > 1 && static_cast<int>(gridDim.x) >= W && me * map.E < N) {
    const int j = blockIdx.x % W;
    const int o = (me + j) % W;
    const int nb = (static_cast<int>(gridDim.x) - j + W - 1) / W;
    const int lo = min(start[o * map.E], rows);
    const int hi = o + 1 < W ? min(start[(o + 1) * map.E], rows) : rows;
    for (int r = lo + static_cast<int>(blockIdx.x / W) * kPermWarps + warp; r < hi; r += nb * kPermWarps) move_row(r);
  } else {
    const int rot = (W > 1 && me * map.E < N && rows > 0) ? min(start[me * map.E], rows) % rows : 0;
    for (int rl = blockIdx.x * kPermWarps + warp; rl < rows; rl += gridDim.x * kPermWarps)
      move_row(rl + rot < rows ? rl + rot : rl + rot - rows);
  }
}

// Zero the padding rows [start + real, start + rows) of each segment in up to two row buffers.
__global__ void zero_pad_rows_kernel(const int* __restrict__ seg_start, const int* __restrict__ seg_rows,
                                     const int* __restrict__ seg_real, int G, __nv_bfloat16* a, int wa,
                                     __nv_bfloat16* b, int wb) {
  const int g = blockIdx.x;
  if (g >= G) return;
  const int r0 = seg_start[g] + seg_real[g], r1 = seg_start[g] + seg_rows[g];
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int r = r0; r < r1; ++r) {
    if (a)
      for (int v = threadIdx.x; v < wa / 8; v += blockDim.x) reinterpret_cast<uint4*>(a + static_cast<long long>(r) * wa)[v] = z;
    if (b)
      for (int v = threadIdx.x; v < wb / 8; v += blockDim.x) reinterpret_cast<uint4*>(b + static_cast<long long>(r) * wb)[v] = z;
  }
}

}  // namespace

void zero_pad_rows(const int* seg_start, const int* seg_rows, const int* seg_real, int G, __nv_bfloat16* a, int wa,
                   __nv_bfloat16* b, int wb, cudaStream_t s) {
  zero_pad_rows_kernel<<<G, 128, 0, s>>>(seg_start, seg_rows, seg_real, G, a, wa, b, wb);
  TAMOE_CUDA(cudaGetLastError());
}

void route_bucket(const RouteDims& d, const RouteBuffers& b, cudaStream_t s, bool direct) {
  launch_pdl(route_scan_kernel, d.N, kScanThreads, 0, s, d, b, direct ? 1 : 0);
  TAMOE_CUDA(cudaGetLastError());
  const size_t smem = sizeof(int) * (5 * d.N + kRouteTile * d.k + 32);
  launch_pdl(route_bucket_kernel, d.tiles(), kRouteTile, smem, s, d, b, direct ? 1 : 0);
  TAMOE_CUDA(cudaGetLastError());
}

void route_capacity(const RouteDims& d, const RouteBuffers& b, int mode, const int* caps, cudaStream_t s) {
  require(mode >= 0 && mode <= 4, "unknown capacity mode");
  launch_pdl(route_capacity_kernel, d.N, kCapThreads, 0, s, d, b, mode, caps);
  TAMOE_CUDA(cudaGetLastError());
}

void route_permute(const RouteDims& d, const RouteBuffers& b, const __nv_bfloat16* x, int dx, const PeerBufs& xp,
                   int r_max, const PeerBufs* zrows, int zdim, const RowMap& map, cudaStream_t s,
                   const PeerInts* codes, int me, int trash_row) {
  require(dx % 8 == 0 && (zrows == nullptr || zdim % 8 == 0), "permute: row widths must be multiples of 8");
  const int blocks = std::max(1, std::min((r_max + kPermWarps - 1) / kPermWarps, 8 * num_sms()));
  const size_t smem = sizeof(int) * (2 * d.N + 32);
  PeerBufs z{};
  if (zrows) z = *zrows;
  PeerInts c{};
  if (codes) c = *codes;
  launch_pdl(route_permute_kernel, blocks, kPermWarps * 32, smem, s, d, b, x, dx, xp, r_max, z, zrows ? 1 : 0, zdim,
             map, c, codes ? 1 : 0, me, trash_row);
  TAMOE_CUDA(cudaGetLastError());
}

}  // namespace tamoe
