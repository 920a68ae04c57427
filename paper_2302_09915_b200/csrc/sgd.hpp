#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace tamoe {

// master -= lr * grad; work = bf16(master)   (trainer.cpp:410-416)
void sgd_step(float* master, const __nv_bfloat16* grad, float lr, __nv_bfloat16* work, long long n, cudaStream_t s);
void sgd_step(float* master, const float* grad, float lr, __nv_bfloat16* work, long long n, cudaStream_t s);
// fp64 weights (reference precision): w -= lr * grad, the product rounded before the subtraction
void sgd_step_f64(double* w, const double* grad, double lr, long long n, cudaStream_t s);
// master = float(w)
void widen_bf16(const __nv_bfloat16* w, float* master, long long n, cudaStream_t s);

}  // namespace tamoe
