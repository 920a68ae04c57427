#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "route.hpp"

namespace tamoe {

// One launch (logits GEMM with the routing in its epilogue) for N <= 64 experts without the fp64 probabilities
// output; otherwise the logits GEMM + the separate router kernel.
bool gate_is_fused(int N, bool want_probs);

// Fused tcgen05 gate: x [P*S x dm] bf16, wg [P x n_pad x dm] bf16 (K-major, pad rows zero).
void gate_forward(const __nv_bfloat16* x, const __nv_bfloat16* wg, int n_pad, const RouteDims& d, int dm,
                  const RowRouteOut& o, cudaStream_t s);

}  // namespace tamoe
