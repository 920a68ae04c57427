// NVLink peer-memory bandwidth microbenchmark (single process, all visible GPUs, peer access enabled):
// copy engine vs SM-driven 16-byte stores / loads with several launch shapes, and the all-to-all
// pattern the expert-parallel layer uses (every GPU writes 1/P of a buffer to every GPU at once).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/p2p_bench scripts/p2p_bench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

template <int U>
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x * U;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = i + static_cast<long long>(u) * blockDim.x;
      v[u] = j < n ? src[j] : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = i + static_cast<long long>(u) * blockDim.x;
      if (j < n) dst[j] = v[u];
    }
  }
}

// all-to-all: GPU g writes chunk j of its source (n/P vectors) into GPU j's destination at slot g
// stagger = 1: GPU g starts at chunk g and walks the peers cyclically (no incast on one receiver)
__global__ void a2a_kernel(const uint4* __restrict__ src, uint4** dsts, int P, int me, long long chunk, int stagger) {
  const long long total = chunk * P;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int j = static_cast<int>((i / chunk + (stagger ? me : 0)) % P);
    const long long o = i % chunk;
    dsts[j][me * chunk + o] = src[i];
  }
}

// Segmented all-to-all: rows of `row_bytes` (2 KB, like a d=1024 bf16 token row), each warp moves `seg` bytes
// of 32 consecutive rows per step (lane-quarter groups of 16 B), i.e. what a GEMM epilogue chunk can push or
// pull.  push = local smem-like source -> peer rows; pull = peer rows -> local.
__global__ void seg_kernel(const uint4* __restrict__ src, uint4** peers, uint4* __restrict__ local, int P, int me,
                           long long rows_per_peer, int seg, int pull) {
  const int lane = threadIdx.x & 31;
  const int per_row = seg / 16;           // 16-byte pieces per row segment
  const int rows_per_inst = 32 / per_row; // rows covered by one warp instruction
  const long long segs_per_row = 2048 / seg;
  const long long total = rows_per_peer * P * segs_per_row;  // (row, segment) units
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  // a warp unit = 32 rows x one segment column
  const long long units = total / 32;
  for (long long u = warp; u < units; u += nwarps) {
    const long long row0 = (u / segs_per_row) * 32;
    const int sc = static_cast<int>(u % segs_per_row);
    const int peer = static_cast<int>((row0 / rows_per_peer) % P);
    for (int r = 0; r < 32; r += rows_per_inst) {
      const long long row = row0 + r + lane / per_row;
      const long long off = (row % rows_per_peer + static_cast<long long>(me) * rows_per_peer) * 128 + sc * per_row + lane % per_row;
      const long long loc = row * 128 + sc * per_row + lane % per_row;
      if (pull) local[loc] = peers[peer][off];
      else peers[peer][off] = src[loc];
    }
  }
}

// All-to-all of 2 KB rows, one warp per row: (a) SM stores, 4 x 16 B per lane; (b) the row staged in shared
// memory and written with one TMA bulk store (cp.async.bulk.global.shared::cta) to the peer address.
template <int MODE>
__global__ void __launch_bounds__(256) rows_a2a_kernel(const uint4* __restrict__ src, uint4** dsts, int P, int me,
                                                       long long rows_per_peer) {
  __shared__ __align__(128) uint4 stage[8][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long total = rows_per_peer * P;
  for (long long r = static_cast<long long>(blockIdx.x) * 8 + warp; r < total; r += static_cast<long long>(gridDim.x) * 8) {
    const int j = static_cast<int>((r / rows_per_peer + me) % P);  // staggered
    const long long o = r % rows_per_peer;
    const uint4* s = src + (j * rows_per_peer + o) * 128;
    uint4* d = dsts[j] + (me * rows_per_peer + o) * 128;
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = s[lane + 32 * u];
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) d[lane + 32 * u] = v[u];
    } else {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 4; ++u) stage[warp][lane + 32 * u] = v[u];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&stage[warp][0]));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 2048;" ::"l"(d), "r"(sa) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  if (MODE == 1 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Row all-to-all as pulls: GPU `me` reads rows [me*rpp, (me+1)*rpp) of every GPU's source into its slot j.
__global__ void __launch_bounds__(256) rows_pull_kernel(uint4** srcs, uint4* __restrict__ dst, int P, int me,
                                                        long long rows_per_peer) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long total = rows_per_peer * P;
  for (long long r = static_cast<long long>(blockIdx.x) * 8 + warp; r < total; r += static_cast<long long>(gridDim.x) * 8) {
    const int j = static_cast<int>((r / rows_per_peer + me) % P);
    const long long o = r % rows_per_peer;
    const uint4* s = srcs[j] + (me * rows_per_peer + o) * 128;
    uint4* d = dst + (j * rows_per_peer + o) * 128;
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = s[lane + 32 * u];
#pragma unroll
    for (int u = 0; u < 4; ++u) d[lane + 32 * u] = v[u];
  }
}

static float time_ms(cudaStream_t s, cudaEvent_t a, cudaEvent_t b) {
  float ms;
  CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

int main() {
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  printf("GPUs: %d\n", ng);
  if (ng < 2) return 0;
  const size_t bytes = 64ull << 20;
  const long long nv = bytes / 16;
  std::vector<uint4*> buf(ng), buf2(ng);
  std::vector<cudaStream_t> st(ng);
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < ng; ++h)
      if (h != g) cudaDeviceEnablePeerAccess(h, 0);
    CK(cudaMalloc(&buf[g], bytes));
    CK(cudaMalloc(&buf2[g], bytes));
    CK(cudaMemset(buf[g], 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
  }
  CK(cudaSetDevice(0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  // 1) copy engine 0 -> 1
  for (int it = 0; it < 2; ++it) {
    CK(cudaEventRecord(a, st[0]));
    CK(cudaMemcpyPeerAsync(buf2[1], 1, buf[0], 0, bytes, st[0]));
    CK(cudaEventRecord(b, st[0]));
    float ms = time_ms(st[0], a, b);
    if (it) printf("copy engine 0->1          : %7.1f GB/s\n", bytes / ms / 1e6);
  }
  // 2) SM stores 0 -> 1 (push) and loads 1 -> 0 (pull), several shapes
  const int grids[] = {148, 296, 592, 1184};
  const int blocks[] = {256, 512, 1024};
  for (int dir = 0; dir < 2; ++dir) {
    for (int gi : grids)
      for (int bi : blocks) {
        float best = 1e9;
        for (int it = 0; it < 3; ++it) {
          CK(cudaEventRecord(a, st[0]));
          if (dir == 0) copy_kernel<4><<<gi, bi, 0, st[0]>>>(buf[0], buf2[1], nv);  // push
          else copy_kernel<4><<<gi, bi, 0, st[0]>>>(buf[1], buf2[0], nv);           // pull
          CK(cudaEventRecord(b, st[0]));
          float ms = time_ms(st[0], a, b);
          if (it && ms < best) best = ms;
        }
        printf("SM %-4s grid %5d block %5d : %7.1f GB/s\n", dir == 0 ? "push" : "pull", gi, bi, bytes / best / 1e6);
      }
  }
  // 3) all-to-all over all GPUs, SM stores, every GPU concurrently (plain order, then staggered)
  for (int stagger = 0; stagger < 2; ++stagger)
  for (int gi : {148, 296, 592, 1184, 2368}) {
    std::vector<uint4**> dptr(ng);
    for (int g = 0; g < ng; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaMalloc(&dptr[g], sizeof(uint4*) * ng));
      CK(cudaMemcpy(dptr[g], buf2.data(), sizeof(uint4*) * ng, cudaMemcpyHostToDevice));
    }
    const long long chunk = nv / ng;
    float worst = 0;
    for (int it = 0; it < 3; ++it) {
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      std::vector<cudaEvent_t> ea(ng), eb(ng);
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventCreate(&ea[g]));
        CK(cudaEventCreate(&eb[g]));
        CK(cudaEventRecord(ea[g], st[g]));
        a2a_kernel<<<gi, 512, 0, st[g]>>>(buf[g], dptr[g], ng, g, chunk, stagger);
        CK(cudaEventRecord(eb[g], st[g]));
      }
      float mx = 0;
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        mx = std::max(mx, time_ms(st[g], ea[g], eb[g]));
      }
      if (it) worst = mx;
    }
    const double off = bytes * (ng - 1.0) / ng;
    printf("a2a %d GPUs %s grid %5d: %7.1f GB/s off-rank per GPU (%.1f us for %zu MiB/GPU)\n", ng,
           stagger ? "staggered" : "in order ", gi,
           off / worst / 1e6, worst * 1e3, bytes >> 20);
  }
  // 3b) row all-to-all: SM stores vs TMA bulk stores
  {
    std::vector<uint4**> dptr(ng);
    for (int g = 0; g < ng; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaMalloc(&dptr[g], sizeof(uint4*) * ng));
      CK(cudaMemcpy(dptr[g], buf2.data(), sizeof(uint4*) * ng, cudaMemcpyHostToDevice));
    }
    const long long rows_per_peer = (bytes / 2048) / ng;
    for (int mode = 0; mode < 2; ++mode)
      for (int gi : {296, 592, 1184, 2368}) {
        float worst = 0;
        for (int it = 0; it < 3; ++it) {
          for (int g = 0; g < ng; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaDeviceSynchronize());
          }
          std::vector<cudaEvent_t> ea(ng), eb(ng);
          for (int g = 0; g < ng; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventCreate(&ea[g]));
            CK(cudaEventCreate(&eb[g]));
            CK(cudaEventRecord(ea[g], st[g]));
            if (mode == 0) rows_a2a_kernel<0><<<gi, 256, 0, st[g]>>>(buf[g], dptr[g], ng, g, rows_per_peer);
            else rows_a2a_kernel<1><<<gi, 256, 0, st[g]>>>(buf[g], dptr[g], ng, g, rows_per_peer);
            CK(cudaEventRecord(eb[g], st[g]));
          }
          float mx = 0;
          for (int g = 0; g < ng; ++g) {
            CK(cudaSetDevice(g));
            mx = std::max(mx, time_ms(st[g], ea[g], eb[g]));
          }
          if (it) worst = mx;
        }
        const double off = bytes * (ng - 1.0) / ng;
        printf("rows a2a %s grid %5d: %7.1f GB/s off-rank per GPU\n", mode ? "TMA bulk" : "SM st  ", gi, off / worst / 1e6);
      }
  }
  // 3c) row all-to-all as pulls (every GPU reads its 1/P slot from every peer) and larger grids
  {
    std::vector<uint4**> sptr(ng);
    for (int g = 0; g < ng; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaMalloc(&sptr[g], sizeof(uint4*) * ng));
      CK(cudaMemcpy(sptr[g], buf.data(), sizeof(uint4*) * ng, cudaMemcpyHostToDevice));
    }
    const long long rows_per_peer = (bytes / 2048) / ng;
    for (int gi : {592, 1184, 2368, 4736}) {
      float worst = 0;
      for (int it = 0; it < 3; ++it) {
        for (int g = 0; g < ng; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaDeviceSynchronize());
        }
        std::vector<cudaEvent_t> ea(ng), eb(ng);
        for (int g = 0; g < ng; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventCreate(&ea[g]));
          CK(cudaEventCreate(&eb[g]));
          CK(cudaEventRecord(ea[g], st[g]));
          rows_pull_kernel<<<gi, 256, 0, st[g]>>>(sptr[g], buf2[g], ng, g, rows_per_peer);
          CK(cudaEventRecord(eb[g], st[g]));
        }
        float mx = 0;
        for (int g = 0; g < ng; ++g) {
          CK(cudaSetDevice(g));
          mx = std::max(mx, time_ms(st[g], ea[g], eb[g]));
        }
        if (it) worst = mx;
      }
      const double off = bytes * (ng - 1.0) / ng;
      printf("rows a2a pull     grid %5d: %7.1f GB/s off-rank per GPU\n", gi, off / worst / 1e6);
    }
  }
  // 3d) all-to-all on the copy engines: every GPU issues P-1 peer copies on P-1 streams at once
  {
    std::vector<std::vector<cudaStream_t>> cs(ng, std::vector<cudaStream_t>(ng));
    for (int g = 0; g < ng; ++g) {
      CK(cudaSetDevice(g));
      for (int j = 0; j < ng; ++j) CK(cudaStreamCreateWithFlags(&cs[g][j], cudaStreamNonBlocking));
    }
    const size_t chunk = bytes / ng;
    float worst = 0;
    for (int it = 0; it < 4; ++it) {
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      std::vector<cudaEvent_t> ea(ng), eb(ng);
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventCreate(&ea[g]));
        CK(cudaEventCreate(&eb[g]));
        CK(cudaEventRecord(ea[g], st[g]));
        for (int j = 0; j < ng; ++j) {
          if (j == g) continue;
          CK(cudaStreamWaitEvent(cs[g][j], ea[g], 0));
          CK(cudaMemcpyPeerAsync(reinterpret_cast<char*>(buf2[j]) + g * chunk, j,
                                 reinterpret_cast<char*>(buf[g]) + j * chunk, g, chunk, cs[g][j]));
          cudaEvent_t ej;
          CK(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
          CK(cudaEventRecord(ej, cs[g][j]));
          CK(cudaStreamWaitEvent(st[g], ej, 0));
        }
        CK(cudaEventRecord(eb[g], st[g]));
      }
      float mx = 0;
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        mx = std::max(mx, time_ms(st[g], ea[g], eb[g]));
      }
      if (it) worst = mx;
    }
    const double off = bytes * (ng - 1.0) / ng;
    printf("a2a copy engines  (%d streams/GPU): %7.1f GB/s off-rank per GPU (%.1f us)\n", ng - 1, off / worst / 1e6,
           worst * 1e3);
  }
  // 4) segmented all-to-all (push / pull), 64 B .. 2 KB segments
  {
    std::vector<uint4**> dptr(ng);
    for (int g = 0; g < ng; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaMalloc(&dptr[g], sizeof(uint4*) * ng));
      CK(cudaMemcpy(dptr[g], buf2.data(), sizeof(uint4*) * ng, cudaMemcpyHostToDevice));
    }
    const long long rows = bytes / 2048;  // rows per GPU buffer
    const long long rows_per_peer = rows / ng;
    for (int pull = 0; pull < 2; ++pull)
      for (int seg : {64, 128, 256, 512, 2048}) {
        float worst = 0;
        for (int it = 0; it < 3; ++it) {
          for (int g = 0; g < ng; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaDeviceSynchronize());
          }
          std::vector<cudaEvent_t> ea(ng), eb(ng);
          for (int g = 0; g < ng; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventCreate(&ea[g]));
            CK(cudaEventCreate(&eb[g]));
            CK(cudaEventRecord(ea[g], st[g]));
            seg_kernel<<<1184, 512, 0, st[g]>>>(buf[g], dptr[g], pull ? buf2[g] : nullptr, ng, g, rows_per_peer,
                                                seg < 512 ? seg : 512, pull);
            CK(cudaEventRecord(eb[g], st[g]));
          }
          float mx = 0;
          for (int g = 0; g < ng; ++g) {
            CK(cudaSetDevice(g));
            mx = std::max(mx, time_ms(st[g], ea[g], eb[g]));
          }
          if (it) worst = mx;
        }
        const double off = bytes * (ng - 1.0) / ng;
        printf("seg a2a %s %4d B segments: %7.1f GB/s off-rank per GPU\n", pull ? "pull" : "push", seg < 512 ? seg : 512,
               off / worst / 1e6);
      }
  }
  return 0;
}
