/*
 * tamoe.h -- C ABI of the B200-native TA-MoE expert-parallel layer.
 *
 * Drop-in boundary for the reference's operator API (namespace tad, C++20,
 * /root/reference/proj/core/include/tadispatch/gate.hpp:22-97 and the inline
 * MoE layer of trainer.cpp:243-356).  Every entry point names the reference
 * symbol it replaces.  Plain pointers and sizes only; device pointers are
 * caller-owned CUDA allocations, `stream` is a cudaStream_t (NULL = legacy).
 *
 * Status codes mirror the reference CLI (tools/main.cpp:435-441):
 *   0 ok, 1 internal (CUDA / NCCL / runtime), 2 validation (tad::ValidationError).
 * tamoe_last_error() returns the message of the last failing call on this thread.
 */
#ifndef TAMOE_H_
#define TAMOE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TAMOE_OK 0
#define TAMOE_ERR_INTERNAL 1
#define TAMOE_ERR_VALIDATION 2

/* Capacity modes: reference CapacityMode (gate.hpp:40). */
#define TAMOE_CAP_NONE 0
#define TAMOE_CAP_GLOBAL 1
#define TAMOE_CAP_LOCAL 2
#define TAMOE_CAP_PROPORTIONAL 3

/* Penalty normalisations: reference PenaltyNorm (gate.hpp:74). */
#define TAMOE_NORM_SUM 0
#define TAMOE_NORM_SOFTMAX 1

/* Expert activation (reference expert is linear: trainer.cpp:284-289). */
#define TAMOE_ACT_NONE 0
#define TAMOE_ACT_GELU 1
#define TAMOE_ACT_RELU 2

/* Aux loss kinds: reference LossKind (trainer.hpp:47). */
#define TAMOE_LOSS_BALANCE 0
#define TAMOE_LOSS_TOPO 1

const char* tamoe_last_error(void);
int tamoe_version(void);

/* ------------------------------------------------------------------ host-side topology inputs
 * Computed once per topology (fp64, host memory, no GPU needed). */

/* largest_remainder_round (gate.cpp:52-78 / gate.hpp:69). out: int64[n]. */
int tamoe_largest_remainder_round(const double* values, int n, long long target, long long* out);

/* penalty_weights (gate.cpp:222-246 / gate.hpp:81). p: double[n]. temperature <= 0 -> mean(1/c_hat). */
int tamoe_penalty_weights(const double* c_hat_row, int n, int norm, double temperature, double* p);

/* target_closed_form (solver.cpp:28-52): Eq. 8, c_hat[P x N] from beta_hat[P x P]. */
int tamoe_target_closed_form(const double* beta_hat, int P, int N, int k, int S, double* c_hat);

/* Capacity per (process, expert) bucket as topk_route derives it (gate.cpp:151-180).
 * caps: int64[P x N]; for TAMOE_CAP_GLOBAL every row holds the single global cap;
 * for TAMOE_CAP_NONE every entry is INT64_MAX.  c_hat (P x N) required for proportional. */
int tamoe_capacity_caps(int mode, double capacity_factor, int k, int S, int N, int P, const double* c_hat,
                        long long* caps);

/* device_payload_tokens (dispatch.cpp:21-26): payload[P x P] = sum of counts[i][e] over experts of j. */
int tamoe_device_payload_tokens(const double* counts, int P, int N, double* payload);

/* ------------------------------------------------------------------ grouped expert GEMMs (device)
 * Building blocks of the expert FFN (trainer.cpp:284-289 / 310-316 generalised).
 * tokens are bf16 [R x K] row-major; group g owns rows [seg_start[g], seg_start[g]+seg_rows[g]),
 * seg_rows multiple of 16 (zero padded).  seg_start / seg_rows are device int32[G]. */
int tamoe_grouped_fwd(const void* tokens, const void* w, int G, int M, int K, int R, const int* seg_start,
                      const int* seg_rows, void* out, void* pre_out, int act, void* stream);
int tamoe_grouped_dgrad(const void* grad_tokens, const void* w, int G, int M, int K, int R, const int* seg_start,
                        const int* seg_rows, void* out, const void* pre_in, int act, void* stream);
int tamoe_grouped_wgrad(const void* a_tokens, const void* b_tokens, int G, int M, int N, int R,
                        const int* seg_start, const int* seg_rows, void* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TAMOE_H_ */
