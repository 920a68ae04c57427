// Device-side expert-parallel plan from the all-gathered counts (one small CTA; P <= 16, N <= 256).
#include <algorithm>

#include "common.hpp"
#include "ep.hpp"
#include "ptx.cuh"

namespace tamoe {

namespace {

__device__ __forceinline__ int pad16(int c) { return (c + 15) & ~15; }

// expert-major receive layouts: at rank j, local expert e_l owns rows
//   [ sum_{e' < e_l} sum_src pad16(c[src][jE+e']) , ... ) split into per-source segments in rank order.
__global__ void ep_plan_kernel(EpPlanDev p, int P, int E, int me) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int N = P * E;
  // one thread per global expert: where do my rows for it start at its owner?
  for (int ge = threadIdx.x; ge < N; ge += blockDim.x) {
    const int j = ge / E, el = ge % E;
    int off = 0;
    for (int e2 = 0; e2 < el; ++e2)
      for (int i = 0; i < P; ++i) off += pad16(p.all_counts[i * N + j * E + e2]);
    for (int i = 0; i < me; ++i) off += pad16(p.all_counts[i * N + ge]);
    p.dst_off[ge] = off;
  }
  if (threadIdx.x == 0) {
    int row = 0;
    for (int el = 0; el < E; ++el) {
      p.seg_start[el] = row;
      for (int i = 0; i < P; ++i) row += pad16(p.all_counts[i * N + me * E + el]);
      p.seg_rows[el] = row - p.seg_start[el];
    }
    *p.recv_rows = row;
  }
}

// Return map of the receive layout: block (local expert el, source i) fills its segment's rows with
// (i, row of the same pick in source i's local layout = expert-major, 16-padded, global expert order).
__global__ void ep_push_map_kernel(EpPlanDev p, int P, int E, int me) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int N = P * E;
  const int el = blockIdx.x / P, i = blockIdx.x % P;
  const int ge = me * E + el;
  __shared__ int s_dst, s_src;
  if (threadIdx.x == 0) {
    int dst = 0;
    for (int e2 = 0; e2 < el; ++e2)
      for (int i2 = 0; i2 < P; ++i2) dst += pad16(p.all_counts[i2 * N + me * E + e2]);
    for (int i2 = 0; i2 < i; ++i2) dst += pad16(p.all_counts[i2 * N + ge]);
    int src = 0;
    for (int e2 = 0; e2 < ge; ++e2) src += pad16(p.all_counts[i * N + e2]);
    s_dst = dst;
    s_src = src;
  }
  __syncthreads();
  const int rows = pad16(p.all_counts[i * N + ge]);
  for (int r = threadIdx.x; r < rows; r += blockDim.x) p.push_row[s_dst + r] = (i << 27) | (s_src + r);
}

__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void ep_barrier_kernel(const __grid_constant__ EpSignal a) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  if (a.my_counts) {
    for (int i = threadIdx.x; i < a.P * a.N; i += blockDim.x) {
      const int r = i / a.N, e = i - r * a.N;
      a.counts_dst[r][a.me * a.N + e] = a.my_counts[e];
    }
  }
  __threadfence_system();  // this kernel's stores (and, by kernel order, earlier kernels') before the signal
  __shared__ unsigned int ep;
  __syncthreads();
  if (threadIdx.x == 0) {
    ep = *a.epoch + 1u;
    *a.epoch = ep;
  }
  __syncthreads();
  const int r = threadIdx.x;
  if (r < a.P) {
    st_release_sys(a.sig[r] + a.me, ep);
    const unsigned int* mine = a.sig[a.me] + r;
    const unsigned long long t0 = global_ns();
    // a peer may already be one barrier ahead (it can only pass `ep` after our signal): compare mod 2^32
    while (static_cast<int>(ld_acquire_sys(mine) - ep) < 0) {
      const unsigned long long dt = global_ns() - t0;
      if (a.soft && dt > 5000000000ull) break;  // teardown: a peer that already exited
      if (dt > 20000000000ull) __trap();
    }
  }
  __syncthreads();
}

// Peer copy of the P2P sweep: 16-byte vectors, 8 per lane in flight, grid of 2 CTAs per SM.
__global__ void __launch_bounds__(512) p2p_copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                       long long n, int rep) {
  constexpr int kU = 8;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x * kU;
  for (long long i0 = static_cast<long long>(blockIdx.x) * blockDim.x * kU + threadIdx.x; i0 < n; i0 += stride) {
    uint4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long i = i0 + static_cast<long long>(u) * blockDim.x;
      if (i < n) v[u] = src[i];
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long i = i0 + static_cast<long long>(u) * blockDim.x;
      if (i < n) dst[i] = v[u];
    }
    if (rep > 1) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const long long i = i0 + static_cast<long long>(u) * blockDim.x;
        if (i < n) store_repeat(dst + i, v[u], rep);
      }
    }
  }
}

__global__ void peer_broadcast_kernel(const __grid_constant__ PeerWords dst, long long off,
                                      const unsigned int* __restrict__ src, long long words, int P) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < words; i += stride) {
    const unsigned int v = src[i];
    for (int r = 0; r < P; ++r) dst.p[r][off + i] = v;
  }
  __threadfence_system();
}

}  // namespace

void peer_broadcast_words(const PeerWords& dst, long long dst_off_words, const void* src, long long words, int P,
                          cudaStream_t s) {
  if (words <= 0) return;
  const int grid = static_cast<int>(std::min<long long>((words + 255) / 256, 2LL * num_sms()));
  launch_pdl(peer_broadcast_kernel, grid, 256, 0, s, dst, dst_off_words, static_cast<const unsigned int*>(src), words, P);
  TAMOE_CUDA(cudaGetLastError());
}

void p2p_copy(void* dst, const void* src, size_t bytes, cudaStream_t s, int rep) {
  require(bytes % 16 == 0, "p2p copy: size must be a multiple of 16 bytes");
  const long long n = static_cast<long long>(bytes / 16);
  const long long per_block = 512LL * 8;
  const int grid = static_cast<int>(std::min<long long>(2LL * num_sms(), (n + per_block - 1) / per_block));
  p2p_copy_kernel<<<std::max(grid, 1), 512, 0, s>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), n,
                                                         rep);
  TAMOE_CUDA(cudaGetLastError());
}

void ep_signal_barrier(const EpSignal& a, cudaStream_t s) {
  launch_pdl(ep_barrier_kernel, 1, 256, 0, s, a);
  TAMOE_CUDA(cudaGetLastError());
}

void ep_plan_device(const EpPlanDev& plan, int P, int E, int me, cudaStream_t s) {
  require(P >= 1 && P <= kMaxRanks, "expert parallelism supports up to 16 ranks");
  launch_pdl(ep_plan_kernel, 1, 128, 0, s, plan, P, E, me);
  TAMOE_CUDA(cudaGetLastError());
  if (plan.push_row) {
    launch_pdl(ep_push_map_kernel, E * P, 128, 0, s, plan, P, E, me);
    TAMOE_CUDA(cudaGetLastError());
  }
}

}  // namespace tamoe
