#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "route.hpp"

namespace tamoe {

enum ActKind : int { kActNone = 0, kActGelu = 1, kActRelu = 2 };

// Expert-parallel return path: instead of storing output row y locally, the epilogue stores it straight
// into the token's home rank (NVLink peer store): row_code[y] = rank << 27 | row in that rank's buffer.
struct SwapPush {
  PeerBufs dst;
  const int* row_code = nullptr;
};

// out[R x M] = act(tokens[seg_g] . W_g^T), W_g = w[g] stored M x K. pre_out (optional) keeps the
// activation derivative act'(pre-activation) for the backward pass.
void grouped_fwd(const __nv_bfloat16* tokens, const __nv_bfloat16* w, int G, int M, int K, int R,
                 const int* seg_start, const int* seg_rows, __nv_bfloat16* out, __nv_bfloat16* pre_out, int act,
                 cudaStream_t s, int w_mod = 0, const SwapPush* push = nullptr);

// out[R x M] = (grad_tokens[seg_g] . W_g) * pre_in, W_g = w[g] stored K x M, pre_in = the act'(pre-activation)
// stored by grouped_fwd (or null).  push (optional, plain outputs only): rows go to their home ranks.
void grouped_dgrad(const __nv_bfloat16* grad_tokens, const __nv_bfloat16* w, int G, int M, int K, int R,
                   const int* seg_start, const int* seg_rows, __nv_bfloat16* out, const __nv_bfloat16* pre_in,
                   int act, cudaStream_t s, int w_mod = 0, const SwapPush* push = nullptr);

// out[g] (M x N) = sum over sub-segments s < nsub of a_tokens[seg_{s*G+g}]^T . b_tokens[seg_{s*G+g}];
// zeros for empty groups.  (w_mod / nsub let expert-parallel receive layouts -- (source, expert)
// segments -- feed the GEMMs without a staging copy.)
void grouped_wgrad(const __nv_bfloat16* a_tokens, const __nv_bfloat16* b_tokens, int G, int M, int N, int R,
                   const int* seg_start, const int* seg_rows, __nv_bfloat16* out, cudaStream_t s, int nsub = 1);

// The FFN's two forward GEMMs (H = act(X W1^T) with act' kept, then O = H W2^T) in one persistent launch: CTAs that
// finish the first GEMM start the second as soon as the H rows of a (group, token tile) are stored.  ready: device
// int [G x chain_ready_stride(R)] scratch (zeroed by the call).  Needs f, d_out multiples of 256 (CTA pairs).
int chain_ready_stride(int R);
void grouped_ffn_fwd_chain(const __nv_bfloat16* tokens, const __nv_bfloat16* w1, const __nv_bfloat16* w2, int G,
                           int f, int d, int d_out, int R, const int* seg_start, const int* seg_rows,
                           __nv_bfloat16* H, __nv_bfloat16* dact, __nv_bfloat16* out, int act, int* ready,
                           cudaStream_t s, int w_mod = 0, const SwapPush* push = nullptr);
// The FFN's two input-gradient GEMMs (dA = (dO W2) * act', then dX = dA W1) in one persistent launch.
void grouped_ffn_dgrad_chain(const __nv_bfloat16* dO, const __nv_bfloat16* w2, const __nv_bfloat16* w1, int G, int f,
                             int d, int d_out, int R, const int* seg_start, const int* seg_rows, __nv_bfloat16* dA,
                             const __nv_bfloat16* dact, __nv_bfloat16* dx_out, int act, int* ready, cudaStream_t s,
                             int w_mod = 0, const SwapPush* push = nullptr);

}  // namespace tamoe
