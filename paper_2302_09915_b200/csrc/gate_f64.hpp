// fp64 device operators in the reference's arithmetic order (see gate_f64.cu).  All pointers are device memory.
#pragma once
#include <cuda_runtime.h>

namespace tamoe {

// c [M x N] = a [M x K] * b [K x N]   (matrix.hpp:83-94, bit-identical)
void matmul_f64(const double* a, const double* b, double* c, int M, int N, int K, cudaStream_t s);
// c [M x N] += a^T b, a [K x M], b [K x N]   (matrix.hpp:96-104 with alpha = 1, bit-identical)
void add_atb_f64(double* c, const double* a, const double* b, int K, int M, int N, cudaStream_t s);
// softmax_rows (gate.cpp:12-28); *bad set to 1 if any logit is non-finite (the row is left unwritten)
void softmax_rows_f64(const double* logits, double* probs, int rows, int cols, int* bad, cudaStream_t s);
// dz = p (coeff - <coeff, p>) per row (gate.cpp:260-266); coeff: device [cols]
void aux_dz_f64(const double* probs, const double* coeff, double* dz, int rows, int cols, cudaStream_t s);

}  // namespace tamoe
