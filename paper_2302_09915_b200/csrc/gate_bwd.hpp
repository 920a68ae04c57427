#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "route.hpp"

namespace tamoe {

struct GateDzArgs {
  int P, S, N, k, n64, dout;
  int P_global;
  int aux_kind;        // 0 balance, 1 topo
  double aux_weight;
  const float* logits;       // [P*S x N]
  const int* idx;            // [P*S*k]
  const double* score;       // [P*S*k]
  const float* dldg;         // [P*S*k]
  const int* counts;         // [P x N] kept
  const double* mean_probs;  // [P x N]
  const double* penalties;   // [P x N]
  const double* loss_part;   // combine partial sums
  int n_loss_part;
  double* losses;            // [2] task (this device's share), aux (this device's share)
  __nv_bfloat16* dz;         // [P*S x n64]
};

inline int expert_pad64(int N) { return N <= 64 ? 64 : (N <= 128 ? 128 : 256); }

void gate_dz(const GateDzArgs& a, cudaStream_t s);
int gate_dw_splits(int P, int S, int d, int n64);
// finalize (optional): the loss finalisation of a gate dz pass that was fused into the combine kernel
void gate_dw(const __nv_bfloat16* x, const __nv_bfloat16* dz, int P, int S, int d, int n64, int n_pad, int N,
             float* part, int splits, float* dwg, cudaStream_t s, const GateDzArgs* finalize = nullptr);
// dX = dz Wg + sum over kept slots of the expert-path gradient rows (read from the owners' layouts).
void gate_dx(const __nv_bfloat16* dz, const __nv_bfloat16* wg, int P, int S, int d, int n64, int n_pad,
             const PeerBufs& dxp, const int* pos, const int* idx, const RowMap& map, int k, __nv_bfloat16* dx,
             cudaStream_t s);

}  // namespace tamoe
