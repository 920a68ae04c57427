// Weighted gather-combine fused with the reference's task loss and the first
// backward step (trainer.cpp:290-316):
//   y_hat_t = sum_{kept slots} g_slot * O[pos(t, slot)]           (combine)
//   r_t     = y_hat_t - y_t ;  task += |r_t|^2                      (MSE)
//   dO[pos] = (2 / (P S d_out)) * g_slot * r_t                       (combine backward, scattered
//                                                                     straight into expert order)
//   dldg    = (2 / (P S d_out)) * <r_t, O[pos]>                      (gate-value gradient)
// One warp per token, 16-byte vectors, fp32 math on bf16 rows.
#include <cuda_bf16.h>

#include "combine.hpp"
#include "common.hpp"
#include "gate_dz.cuh"
#include "ptx.cuh"
#include "route.hpp"

namespace tamoe {

namespace {

constexpr int kCombWarps = 4;

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return v;
}

// KT = compile-time top-k (0: runtime k <= kMaxTopK).  Each lane keeps kU 16-byte vectors of every
// slot in flight before computing, so the warp has (k + 1) * kU * 512 B of loads outstanding.
// NPL > 0: the gate dz pass is fused in (experts per lane, N <= 32 * NPL).
template <int KT, int NPL>
__global__ void __launch_bounds__(kCombWarps * 32) combine_loss_kernel(const __grid_constant__ CombineArgs a) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  constexpr int KM = KT > 0 ? KT : kMaxTopK;
  constexpr int kU = 4;
  __shared__ double wsum[kCombWarps];
  extern __shared__ double coeff[];  // [P*N] aux-loss coefficients (fused dz)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t = static_cast<long long>(blockIdx.x) * kCombWarps + warp;
  if constexpr (NPL > 0) {
    dz_coeff_smem(a.gz, coeff);
    __syncthreads();
  }
  double lsum = 0.0;
  if (t < a.T) {
    const int k = KT > 0 ? KT : a.k;
    float lg[NPL > 0 ? NPL : 1];
    int ex_in[KM];
    double sc_in[KM];
    if constexpr (NPL > 0) {  // the dz pass's inputs, loaded up front so their latency overlaps the combine
      dz_load_logits<NPL>(a.gz, t, lane, lg);
#pragma unroll
      for (int j = 0; j < KM; ++j) {
        ex_in[j] = j < k ? a.idx[t * k + j] : -1;
        sc_in[j] = (k > 1 && j < k) ? a.gz.score[t * k + j] : 0.0;
      }
    }
    int rows[KM];
    float g[KM], dot[KM];
    const __nv_bfloat16* osrc[KM];
    __nv_bfloat16* odst[KM];
    int orep[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      rows[j] = (j < k) ? a.pos[t * k + j] : -1;
      g[j] = (j < k) ? a.gate[t * k + j] : 0.f;
      dot[j] = 0.f;
      // o_home: the expert output of pick t*k+j sits at that row of this rank (its address does not wait
      // for pos; a dropped pick's row is stale and is zeroed after the load)
      osrc[j] = (a.o_home && j < k) ? a.O.p[0] + (t * k + j) * a.dout : nullptr;
      odst[j] = nullptr;
      orep[j] = 1;
      if (rows[j] >= 0) {
        const int ex = a.idx[t * k + j];
        const int owner = a.map.rank_of(ex);
        const long long r = a.map.row(rows[j], ex);
        if (!a.o_home) osrc[j] = a.O.p[owner] + r * a.dout;
        odst[j] = a.dO.p[owner] + r * a.dout;
        orep[j] = a.dO.rep[owner];
      }
    }
    const int nv = a.dout / 8;
    const uint4* __restrict__ y4 = reinterpret_cast<const uint4*>(a.y + t * a.dout);
    for (int v0 = lane; v0 < nv; v0 += 32 * kU) {
      uint4 yv[kU], ov[KM][kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int v = v0 + 32 * u;
        yv[u] = v < nv ? y4[v] : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          ov[j][u] = (osrc[j] && v < nv) ? reinterpret_cast<const uint4*>(osrc[j])[v] : make_uint4(0, 0, 0, 0);
          if (rows[j] < 0) ov[j][u] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int v = v0 + 32 * u;
        if (v >= nv) break;
        float yh[8], o[KM][8];
#pragma unroll
        for (int i = 0; i < 8; ++i) yh[i] = 0.f;
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          unpack8(ov[j][u], o[j]);
#pragma unroll
          for (int i = 0; i < 8; ++i) yh[i] += g[j] * o[j][i];  // dropped slots hold zeros
        }
        if (a.y_hat) reinterpret_cast<uint4*>(a.y_hat + t * a.dout)[v] = pack8(yh);
        float yy[8], r[8];
        unpack8(yv[u], yy);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          r[i] = yh[i] - yy[i];
          lsum += static_cast<double>(r[i]) * r[i];
        }
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          if (rows[j] >= 0) {
            float go[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              dot[j] += r[i] * o[j][i];
              go[i] = a.mse_scale * g[j] * r[i];
            }
            const uint4 gv = pack8(go);
            reinterpret_cast<uint4*>(odst[j])[v] = gv;
            if (orep[j] > 1) store_repeat(reinterpret_cast<uint4*>(odst[j]) + v, gv, orep[j]);
          }
        }
      }
    }
    float dl[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      dl[j] = 0.f;
      if (j < k) {
        float s = dot[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        dl[j] = rows[j] >= 0 ? a.mse_scale * s : 0.f;
        if (lane == 0) a.dldg[t * k + j] = dl[j];
      }
    }
    if constexpr (NPL > 0) dz_token<KM, NPL>(a.gz, coeff, t, k, lane, lg, ex_in, dl, sc_in);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  if (lane == 0) wsum[warp] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kCombWarps; ++w) s += wsum[w];
    a.loss_part[blockIdx.x] = s;
  }
}

}  // namespace

int combine_blocks(long long T) { return static_cast<int>((T + kCombWarps - 1) / kCombWarps); }

template <int KT>
static void launch_combine(const CombineArgs& a, int blocks, cudaStream_t s) {
  if (!a.fuse_dz) {
    launch_pdl(combine_loss_kernel<KT, 0>, blocks, kCombWarps * 32, 0, s, a);
    return;
  }
  const size_t smem = sizeof(double) * a.gz.P * a.gz.N;
  const int N = a.gz.N;
  if (N <= 32) launch_pdl(combine_loss_kernel<KT, 1>, blocks, kCombWarps * 32, smem, s, a);
  else if (N <= 64) launch_pdl(combine_loss_kernel<KT, 2>, blocks, kCombWarps * 32, smem, s, a);
  else if (N <= 128) launch_pdl(combine_loss_kernel<KT, 4>, blocks, kCombWarps * 32, smem, s, a);
  else launch_pdl(combine_loss_kernel<KT, 8>, blocks, kCombWarps * 32, smem, s, a);
}

void combine_loss(const CombineArgs& a, cudaStream_t s) {
  require(a.dout % 8 == 0, "combine: d_out must be a multiple of 8");
  require(a.k >= 1 && a.k <= kMaxTopK, "combine: k out of range");
  require(!a.fuse_dz || (a.gz.N <= 256 && a.gz.P * a.gz.N <= 4096), "combine: fused dz needs N <= 256");
  const int blocks = combine_blocks(a.T);
  if (a.k == 1) launch_combine<1>(a, blocks, s);
  else if (a.k == 2) launch_combine<2>(a, blocks, s);
  else launch_combine<0>(a, blocks, s);
  TAMOE_CUDA(cudaGetLastError());
}

}  // namespace tamoe
