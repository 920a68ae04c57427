#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gate_bwd.hpp"
#include "route.hpp"

namespace tamoe {

struct CombineArgs {
  long long T;  // tokens on this device (P_local * S)
  int k, dout;
  float mse_scale;               // 2 / (P_global * S * d_out), trainer.cpp:243
  const int* pos;                // [T*k] row in this rank's padded expert-major layout (-1 dropped)
  const int* idx;                // [T*k] expert of the pick (owner rank = idx / E)
  const float* gate;             // [T*k]
  PeerBufs O;                    // expert outputs in every owner's receive layout (peer-mapped) ...
  int o_home;                    // ... or (1) already returned into this rank's layout: O.p[0][pos]
  const __nv_bfloat16* y;        // [T x dout] targets
  __nv_bfloat16* y_hat;          // optional [T x dout]
  PeerBufs dO;                   // gradient w.r.t. expert outputs, written into the owner's receive layout
  RowMap map;
  float* dldg;                   // [T*k]
  double* loss_part;             // [combine_blocks(T)] sum of squared residuals per block
  // fuse_dz: the gate's softmax backward (gate_dz) runs per token right after the combine, in the same warp
  // (the loss finalisation then moves into the gate dW GEMM); gz.dldg is not read
  int fuse_dz;
  GateDzArgs gz;
};

int combine_blocks(long long T);
void combine_loss(const CombineArgs& a, cudaStream_t s);

}  // namespace tamoe
