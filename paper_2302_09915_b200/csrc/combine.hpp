#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace tamoe {

struct CombineArgs {
  long long T;  // tokens on this device (P_local * S)
  int k, dout;
  float mse_scale;               // 2 / (P_global * S * d_out), trainer.cpp:243
  const int* pos;                // [T*k] row in the expert-sorted buffer (-1 dropped)
  const float* gate;             // [T*k]
  const __nv_bfloat16* O;        // [R x dout] expert outputs, expert order
  const __nv_bfloat16* y;        // [T x dout] targets
  __nv_bfloat16* y_hat;          // optional [T x dout]
  __nv_bfloat16* dO;             // [R x dout] gradient w.r.t. expert outputs (expert order)
  float* dldg;                   // [T*k]
  double* loss_part;             // [combine_blocks(T)] sum of squared residuals per block
};

int combine_blocks(long long T);
void combine_loss(const CombineArgs& a, cudaStream_t s);

}  // namespace tamoe
