// fp64 gate operators for the reference's value-semantics API (tad::Matrix in, fp64 out), on the device.
//
// The reference's gate is fp64 end to end (matrix.hpp:10-12).  These kernels serve the drop-in C++ shim
// (integration/tad_gate_b200.cpp) that replaces gate.cpp for existing callers, so they reproduce the
// reference's arithmetic order exactly rather than chasing throughput (the layer's hot path is the bf16
// tcgen05 gate in gate.cu):
//   matmul   (matrix.hpp:83-94):  c(i,j) = sum over k ascending of a(i,k)*b(k,j), skipping a(i,k) == 0,
//                                 product rounded before the add (the reference is built without FMA)
//   add_atb  (matrix.hpp:96-104): c(i,j) += sum over k ascending of a(k,i)*b(k,j), skipping a(k,i) == 0
//   softmax_rows (gate.cpp:12-28): max, exp(v - max), sequential sum in expert order, divide
//   grad_aux_loss (gate.cpp:257-271): dot = sum_e coeff_e p_se (expert order), dz = p (coeff - dot), xT dz
// With __dmul_rn / __dadd_rn the matmul and add_atb results are bit-identical to the reference; exp is
// CUDA's (<= 1 ulp, like glibc's), so probabilities can differ from the CPU in the last ulp.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "common.hpp"
#include "gate_f64.hpp"

namespace tamoe {
namespace {

constexpr int kTile = 16;

// C[M x N] (+)= op(A) B with op(A) = A [M x K] (trans = 0) or A^T, A [K x M] (trans = 1).  One thread per
// output element walks k in ascending order; operands are staged through shared memory in 16 x 16 tiles.
__global__ void matmul_f64_kernel(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ c,
                                  int M, int N, int K, int trans, int accumulate) {
  __shared__ double as[kTile][kTile + 1];
  __shared__ double bs[kTile][kTile + 1];
  const int i = blockIdx.y * kTile + threadIdx.y;
  const int j = blockIdx.x * kTile + threadIdx.x;
  double acc = (accumulate && i < M && j < N) ? c[static_cast<long long>(i) * N + j] : 0.0;
  for (int k0 = 0; k0 < K; k0 += kTile) {
    // as[r][kk] = op(A)(blockIdx.y*16 + r, k0 + kk)
    {
      const int r = threadIdx.y, kk = threadIdx.x;
      const int gi = blockIdx.y * kTile + r, gk = k0 + kk;
      double v = 0.0;
      if (gi < M && gk < K) v = trans ? a[static_cast<long long>(gk) * M + gi] : a[static_cast<long long>(gi) * K + gk];
      as[r][kk] = v;
    }
    {
      const int kk = threadIdx.y, col = threadIdx.x;
      const int gk = k0 + kk, gj = blockIdx.x * kTile + col;
      bs[kk][col] = (gk < K && gj < N) ? b[static_cast<long long>(gk) * N + gj] : 0.0;
    }
    __syncthreads();
    const int kend = min(kTile, K - k0);
    for (int kk = 0; kk < kend; ++kk) {
      const double av = as[threadIdx.y][kk];
      if (av != 0.0) acc = __dadd_rn(acc, __dmul_rn(av, bs[kk][threadIdx.x]));
    }
    __syncthreads();
  }
  if (i < M && j < N) c[static_cast<long long>(i) * N + j] = acc;
}

// One thread per row (the reference's per-row loops are sequential in expert order).
__global__ void softmax_rows_f64_kernel(const double* logits, double* probs, int rows,  // may alias
                                        int cols, int* __restrict__ bad) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= rows) return;
  const double* z = logits + static_cast<long long>(s) * cols;
  double* p = probs + static_cast<long long>(s) * cols;
  double mx = -CUDART_INF;
  for (int e = 0; e < cols; ++e) {
    const double v = z[e];
    if (!isfinite(v)) {
      atomicExch(bad, 1);
      return;
    }
    mx = fmax(mx, v);
  }
  double denom = 0.0;
  for (int e = 0; e < cols; ++e) {
    const double v = exp(__dadd_rn(z[e], -mx));
    p[e] = v;
    denom = __dadd_rn(denom, v);
  }
  for (int e = 0; e < cols; ++e) p[e] = __ddiv_rn(p[e], denom);
}

__global__ void aux_dz_f64_kernel(const double* __restrict__ probs, const double* __restrict__ coeff,
                                  double* __restrict__ dz, int rows, int cols) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= rows) return;
  const double* p = probs + static_cast<long long>(s) * cols;
  double* g = dz + static_cast<long long>(s) * cols;
  double dot = 0.0;
  for (int e = 0; e < cols; ++e) dot = __dadd_rn(dot, __dmul_rn(coeff[e], p[e]));
  for (int e = 0; e < cols; ++e) g[e] = __dmul_rn(p[e], __dadd_rn(coeff[e], -dot));
}

void launch_matmul(const double* a, const double* b, double* c, int M, int N, int K, int trans, int acc,
                   cudaStream_t s) {
  if (M == 0 || N == 0) return;
  const dim3 grid((N + kTile - 1) / kTile, (M + kTile - 1) / kTile);
  matmul_f64_kernel<<<grid, dim3(kTile, kTile), 0, s>>>(a, b, c, M, N, K, trans, acc);
  TAMOE_CUDA(cudaGetLastError());
}

}  // namespace

void matmul_f64(const double* a, const double* b, double* c, int M, int N, int K, cudaStream_t s) {
  launch_matmul(a, b, c, M, N, K, 0, 0, s);
}

void add_atb_f64(double* c, const double* a, const double* b, int K, int M, int N, cudaStream_t s) {
  launch_matmul(a, b, c, M, N, K, 1, 1, s);
}

void softmax_rows_f64(const double* logits, double* probs, int rows, int cols, int* bad, cudaStream_t s) {
  if (rows == 0 || cols == 0) return;
  softmax_rows_f64_kernel<<<(rows + 127) / 128, 128, 0, s>>>(logits, probs, rows, cols, bad);
  TAMOE_CUDA(cudaGetLastError());
}

void aux_dz_f64(const double* probs, const double* coeff, double* dz, int rows, int cols, cudaStream_t s) {
  if (rows == 0 || cols == 0) return;
  aux_dz_f64_kernel<<<(rows + 127) / 128, 128, 0, s>>>(probs, coeff, dz, rows, cols);
  TAMOE_CUDA(cudaGetLastError());
}

}  // namespace tamoe
