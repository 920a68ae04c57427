// Plain SGD of train() (trainer.cpp:410-416) on fp32 master weights, with the bf16 working copy the tcgen05
// GEMMs read refreshed in the same pass (an update below half a bf16 ulp would otherwise be lost).
#include <cuda_bf16.h>

#include "common.hpp"
#include "sgd.hpp"

namespace tamoe {

namespace {

template <class G>
__device__ __forceinline__ float to_f(G g) {
  return static_cast<float>(g);
}
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 g) {
  return __bfloat162float(g);
}

template <class G>
__global__ void sgd_kernel(float* __restrict__ master, const G* __restrict__ grad, float lr,
                           __nv_bfloat16* __restrict__ work, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float w = master[i] - lr * to_f(grad[i]);
    master[i] = w;
    work[i] = __float2bfloat16(w);
  }
}

__global__ void widen_kernel(const __nv_bfloat16* __restrict__ w, float* __restrict__ master, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    master[i] = __bfloat162float(w[i]);
}

// fp64 weights in the reference's rounding: w -= (lr * g), product rounded first (no FMA)
__global__ void sgd_f64_kernel(double* __restrict__ w, const double* __restrict__ grad, double lr, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    w[i] = __dsub_rn(w[i], __dmul_rn(lr, grad[i]));
}

int grid_for(long long n) {
  const long long b = (n + 255) / 256;
  return static_cast<int>(b < 4LL * num_sms() ? (b > 0 ? b : 1) : 4LL * num_sms());
}

}  // namespace

void sgd_step(float* master, const __nv_bfloat16* grad, float lr, __nv_bfloat16* work, long long n, cudaStream_t s) {
  sgd_kernel<<<grid_for(n), 256, 0, s>>>(master, grad, lr, work, n);
  TAMOE_CUDA(cudaGetLastError());
}

void sgd_step(float* master, const float* grad, float lr, __nv_bfloat16* work, long long n, cudaStream_t s) {
  sgd_kernel<<<grid_for(n), 256, 0, s>>>(master, grad, lr, work, n);
  TAMOE_CUDA(cudaGetLastError());
}

void sgd_step_f64(double* w, const double* grad, double lr, long long n, cudaStream_t s) {
  if (n <= 0) return;
  sgd_f64_kernel<<<grid_for(n), 256, 0, s>>>(w, grad, lr, n);
  TAMOE_CUDA(cudaGetLastError());
}

void widen_bf16(const __nv_bfloat16* w, float* master, long long n, cudaStream_t s) {
  widen_kernel<<<grid_for(n), 256, 0, s>>>(w, master, n);
  TAMOE_CUDA(cudaGetLastError());
}

}  // namespace tamoe
