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

/* ------------------------------------------------------------------ measured-topology pipeline (host)
 * Symmetric switch trees are passed as their level vector, root first: {8} = one switch, {2,4} = two
 * groups of four (topology.hpp:28-33).  n_levels = 0 means "no topology".  Matrices are P x P row-major,
 * alpha in us, beta in us per decimal MB; NaN marks an unmeasured link. */

/* fit_profile (comm_cost.cpp:57-104 / comm_cost.hpp:44-50): per ordered pair least squares
 * time_us = alpha + beta * message_mb over its samples (TransferSample, profile_io.hpp:8-13). */
int tamoe_fit_profile(const int* src, const int* dst, const double* message_mb, const double* time_us, int n,
                      int P, double* alpha, double* beta);

/* fill_partial_profile (profile.cpp:164-233 / profile.hpp:47-52). */
int tamoe_fill_partial_profile(const double* alpha, const double* beta, int P, const int* levels, int n_levels,
                               double self_beta_floor, double* alpha_out, double* beta_out);

/* smooth_profile (profile.cpp:46-98 / profile.hpp:33): level means over a symmetric tree -> alpha_hat,
 * beta_hat (P x P); level_alpha / level_beta (optional, n_levels entries: one per switch-distance group). */
int tamoe_smooth_profile(const int* levels, int n_levels, const double* alpha, const double* beta, int P,
                         double self_beta_floor, double* alpha_hat, double* beta_hat, double* level_alpha,
                         double* level_beta);

/* NVLink point-to-point sweep (device, collective over `world` processes, one GPU each; the caller has
 * selected its device).  Every ordered pair (src, dst) incl. src == dst and every message size is timed
 * `reps` times (after `warmup`) as one SM-driven peer copy, CUDA events on the source rank.
 * time_us[src][dst][size][rep] is filled on every rank -> TransferSample rows for tamoe_fit_profile. */
int tamoe_p2p_sweep(const void* nccl_id128, int world, int rank, const double* sizes_mb, int nsizes, int reps,
                    int warmup, double* time_us);

/* The same sweep with the external (NCCL-free) bootstrap of tamoe_layer_create_ep_begin: create, exchange
 * the blobs, connect, sweep.  time_us is filled for the rows this rank timed (src == rank), zero elsewhere:
 * the caller sums the ranks' arrays. */
typedef struct tamoe_p2p_probe tamoe_p2p_probe;
int tamoe_p2p_probe_create(int world, int rank, double max_mb, tamoe_p2p_probe** out, void* blob_out);
int tamoe_p2p_probe_connect(tamoe_p2p_probe* p, const void* blobs, int world);
int tamoe_p2p_probe_sweep(tamoe_p2p_probe* p, const double* sizes_mb, int nsizes, int reps, int warmup,
                          double* time_us);
int tamoe_p2p_probe_destroy(tamoe_p2p_probe* p);

/* Heterogeneous-topology emulation (BASELINE config 5): ranks in different groups of `group_size` consecutive
 * ranks exchange over a link throttled `repeat` times -- every payload store to such a peer (dispatch, expert
 * output return, dO, dX return, and the p2p sweep's copies) is issued `repeat` times, so the link delivers
 * 1/repeat of its bandwidth.  Process-wide; applies to layers / sweeps created afterwards.  (0, 1) = off. */
int tamoe_set_link_emulation(int group_size, int repeat);

/* exchange_cost (comm_cost.cpp:24-55): c = dispatch matrix [P x N] tokens, payload d * b bytes per token.
 * pair_cost_us[P x P] (optional); summary[4] = bottleneck_us, total_bytes, size_exchange_us, total_estimate_us. */
int tamoe_exchange_cost(const double* alpha, const double* beta, const double* c, int P, int N, int d, int b,
                        int extra_alpha_rounds, double* pair_cost_us, double* summary);

/* ------------------------------------------------------------------ grouped expert GEMMs (device)
 * Building blocks of the expert FFN (trainer.cpp:284-289 / 310-316 generalised).
 * tokens are bf16 [R x K] row-major; group g owns rows [seg_start[g], seg_start[g]+seg_rows[g]),
 * seg_rows multiple of 16 (zero padded).  seg_start / seg_rows are device int32[G], 1 <= G <= 256.
 * grouped_fwd: out = act(tokens W_g^T), pre_out (optional) = act'(tokens W_g^T) kept for the backward;
 * grouped_dgrad: out = (grad_tokens W_g) * pre_in (elementwise; pre_in = that act', optional). */
int tamoe_grouped_fwd(const void* tokens, const void* w, int G, int M, int K, int R, const int* seg_start,
                      const int* seg_rows, void* out, void* pre_out, int act, void* stream);
int tamoe_grouped_dgrad(const void* grad_tokens, const void* w, int G, int M, int K, int R, const int* seg_start,
                        const int* seg_rows, void* out, const void* pre_in, int act, void* stream);
int tamoe_grouped_wgrad(const void* a_tokens, const void* b_tokens, int G, int M, int N, int R,
                        const int* seg_start, const int* seg_rows, void* out, void* stream);

/* ------------------------------------------------------------------ device router
 * The reference's routing operators on the device: gate_forward (gate.cpp:30-32) and topk_route
 * (gate.cpp:91-202) for P logical processes of S tokens, N experts, top-k (k <= 8). */
typedef struct tamoe_router tamoe_router;

/* Readable routing arrays (tamoe_router_read / tamoe_layer_read). */
#define TAMOE_R_IDX 0         /* int32  [P*S*k] expert of each pick (pick = token*k + slot) */
#define TAMOE_R_GATE 1        /* fp32   [P*S*k] combine weight (gate_value) */
#define TAMOE_R_SCORE 2       /* fp64   [P*S*k] raw selection probability */
#define TAMOE_R_KEPT 3        /* uint8  [P*S*k] */
#define TAMOE_R_POS 4         /* int32  [P*S*k] row in the expert-sorted buffer, -1 if dropped */
#define TAMOE_R_COUNTS 5      /* int32  [P*N] kept per (process, expert) */
#define TAMOE_R_DROPPED 6     /* int32  [P*N] */
#define TAMOE_R_MEAN_PROBS 7  /* fp64   [P*N] column means of the softmax */
#define TAMOE_R_SEG_START 8   /* int32  [N] padded row segment of each expert */
#define TAMOE_R_SEG_ROWS 9    /* int32  [N] */
#define TAMOE_R_CLIST 10      /* int32  [P*S*k] kept picks, expert-major, (process, token) order */
#define TAMOE_R_LIST_START 11 /* int32  [N] start of each expert's range in CLIST */
#define TAMOE_R_BAD 12        /* int32  [1] non-zero if a gate logit was non-finite */
#define TAMOE_R_LOGITS 13     /* fp32   [P*S*N] (layer only) */
#define TAMOE_R_GATE64 14     /* fp64   [P*S*k] gate_value in the reference's fp64 (standalone router only) */

int tamoe_router_create(int P, int S, int N, int k, tamoe_router** out);
int tamoe_router_destroy(tamoe_router* r);
/* topk_route on device fp64 probabilities [P*S*N]; caps = tamoe_capacity_caps() output (host int64 [P*N]). */
int tamoe_router_route_probs(tamoe_router* r, const double* probs, int mode, const long long* caps, void* stream);
/* gate_forward + topk_route fused: x bf16 [P*S x d], wg bf16 [P x n_pad x d] (n_pad = round_up(N,16), pad rows 0).
 * logits (fp32 [P*S x N]) and probs (fp64 [P*S x N]) are optional device outputs.  Raises status 2 on a
 * non-finite logit (gate.cpp:16). */
int tamoe_router_route_gate(tamoe_router* r, const void* x, const void* wg, int n_pad, int d, float* logits,
                            double* probs, int mode, const long long* caps, void* stream);
/* Gather token rows into the padded expert-sorted buffer xp [r_max x d] (pad rows zeroed). */
int tamoe_router_permute(tamoe_router* r, const void* x, int d, void* xp, int r_max, void* stream);
/* Copy a routing array (TAMOE_R_*) to host or device memory; synchronises the stream. */
int tamoe_router_read(tamoe_router* r, int what, void* dst, long long bytes, void* stream);

/* ------------------------------------------------------------------ fp64 value-semantics gate operators
 * The reference's gate API is fp64 (tad::Matrix, matrix.hpp:10-12).  These device entry points serve
 * callers that keep that API (the drop-in shim integration/tad_gate_b200.cpp replacing gate.cpp) and follow
 * the reference's arithmetic order: the matmuls are bit-identical (k ascending, zero skip, no FMA), exp is
 * CUDA's (<= 1 ulp).  Device pointers, row-major; they synchronise `stream` only where a status depends on
 * device data (non-finite logits). */

/* softmax_rows (gate.cpp:12-28): probs [rows x cols]; may alias logits.  Status 2 on a non-finite logit. */
int tamoe_softmax_rows_f64(const double* logits, int rows, int cols, double* probs, void* stream);
/* gate_forward (gate.cpp:30-32): probs [S x N] = softmax_rows(x [S x d] * W [d x N]). */
int tamoe_gate_forward_f64(const double* x, const double* w, int S, int d, int N, double* probs, void* stream);
/* grad_aux_loss (gate.cpp:257-271): grad [d x N] = x^T dz, dz = p (coeff - <coeff, p>) row-wise;
 * coeff is a HOST fp64 [N] vector (tamoe_aux_coefficients). */
int tamoe_grad_aux_loss_f64(const double* x, const double* probs, const double* coeff, int S, int d, int N,
                            double* grad, void* stream);

/* One reference-precision MoE layer step: BASELINE config 1 (fp64, linear experts) on the device.  Replaces the
 * inline step of train() (trainer.cpp:246-356): fp64 gate_forward per process -> topk_route on router r
 * (created with P, S, N, k) -> expert x U_e -> combine -> MSE -> backward (dL/dg, top-k Jacobian, aux
 * coefficients, softmax backward, x^T dz).  Sums run in the reference's order without FMA, so gradients are
 * bit-identical to the reference's whenever the softmax is.  Device fp64, row-major: x [P*S x d],
 * y [P*S x d_out], gates [P x d x N], experts [N x d x d_out]; outputs gate_grads [P x d x N],
 * expert_grads [N x d x d_out], optional probs [P*S x N] and y_hat [P*S x d_out].  Host: penalty [P x N]
 * (topo loss; NULL otherwise), c_hat [P x N] (aux_kind 2 = compulsory quota routing, apply_compulsory_quota
 * trainer.cpp:121-169, top-1 only; NULL otherwise), caps [P x N] (tamoe_capacity_caps), losses [2] = task, aux
 * (TrainReport).  Routing arrays stay readable through tamoe_router_read.  Status 2 on a non-finite logit or
 * an unknown aux kind; status 1 when the step diverges (trainer.cpp:362-366). */
int tamoe_layer_step_f64(tamoe_router* r, int d, int d_out, const double* x, const double* y, const double* gates,
                         const double* experts, const double* penalty, const double* c_hat, int aux_kind,
                         double aux_weight, int cap_mode, const long long* caps, double* probs, double* gate_grads,
                         double* expert_grads, double* y_hat, double* losses, void* stream);

/* Auxiliary losses on a routing result (host, N-vectors; counts int64 = RoutingResult::counts). */
/* loss_balance (gate.cpp:209-214) */
int tamoe_loss_balance(const long long* counts, const double* mean_probs, int N, int S, double* loss);
/* loss_topo (gate.cpp:248-255): N * P * sum over the n = counts.size() entries; penalty [n] */
int tamoe_loss_topo(const long long* counts, const double* mean_probs, const double* penalty, int n, int N, int P,
                    int S, double* loss);
/* balance_coefficients / topo_coefficients (gate.cpp:273-287) over n = counts.size() entries, scaled by
 * N * P (topo): kind TAMOE_LOSS_BALANCE (penalty, N, P unused) or TAMOE_LOSS_TOPO. */
int tamoe_aux_coefficients(int kind, const long long* counts, const double* penalty, int n, int N, int P, int S,
                           double* coeff);

/* ------------------------------------------------------------------ the MoE layer (trainer.cpp:243-356)
 * One step = gate -> route (capacity) -> permute -> experts -> combine -> task MSE + aux loss ->
 * backward (expert dgrad/wgrad, combine-weight Jacobian, softmax backward, dWg, optional dX).
 * No optimizer update (the reference's SGD, trainer.cpp:410-416, is the caller's). */
typedef struct tamoe_layer tamoe_layer;

typedef struct {
  int P;          /* logical processes on this device (reference P when world_size == 1) */
  int S;          /* tokens per process */
  int d, d_out;   /* d % 256 == 0, d_out % 128 == 0 */
  int N, k;       /* experts (<= 256), top-k (<= 8) */
  int f;          /* 0: linear expert U_e (reference); > 0: FFN d -> f -> d_out, f % 256 == 0 */
  int act;        /* TAMOE_ACT_* (FFN only) */
  int cap_mode;   /* TAMOE_CAP_* */
  double capacity_factor;
  int aux_kind;   /* TAMOE_LOSS_* */
  double aux_weight;
  int penalty_norm;
  double temperature;
  int need_dx;    /* compute dL/dx (not in the reference) */
  int world_size, rank;
} tamoe_layer_config;

typedef struct {
  const void* x;   /* bf16 [P*S x d] */
  const void* y;   /* bf16 [P*S x d_out] regression targets (trainer.cpp:290-296) */
  const void* wg;  /* bf16 [P x n_pad x d] gate weights (reference W_i transposed, pad rows zero) */
  const void* w1;  /* linear: bf16 [E x d_out x d] = U_e^T;  FFN: bf16 [E x f x d] */
  const void* w2;  /* FFN: bf16 [E x d_out x f] */
  float* dwg;      /* fp32 [P x n_pad x d] */
  void* dw1;       /* bf16, shape of w1 */
  void* dw2;       /* bf16, shape of w2 */
  void* dx;        /* bf16 [P*S x d] when need_dx */
  void* y_hat;     /* optional bf16 [P*S x d_out] */
  double* losses;  /* device fp64[2]: task MSE, aux loss (this device's share) */
} tamoe_layer_io;

/* c_hat: host fp64 [P_global x N] dispatch target (required for topo loss / proportional capacity). */
int tamoe_layer_create(const tamoe_layer_config* cfg, const double* c_hat, tamoe_layer** out);

/* Expert parallelism across GPUs (one process per GPU, NVLink / NVSwitch).
 * Rank r owns experts [r*E, (r+1)*E), E = N / world_size (dispatch.hpp:31); gate replicas are per rank with
 * no all-reduce (trainer.cpp:207-216).  Ranks map each other's workspaces (CUDA IPC) and every payload is a
 * peer store from the kernel that computes it: the permute kernel stores token rows into the owners
 * (dispatch), the owners' fwd2 / dgrad1 GEMM epilogues store expert outputs / input gradients back into the
 * tokens' home ranks, the combine kernel stores dO into the owners; phases are ordered by a device-side
 * barrier over the mapped workspaces that also carries the counts all-gather (NCCL is used at setup only).
 * Local / proportional capacities are rank-local (gate.cpp:165-180); global capacity across ranks adds a picks
 * exchange into every rank's global view (gate.cpp:157-164).  tamoe_nccl_unique_id fills 128 bytes on one rank; broadcast them to all ranks, then
 * every rank calls tamoe_layer_create_ep with its cfg.rank / cfg.world_size. */
int tamoe_nccl_unique_id(void* out128);
int tamoe_layer_create_ep(const tamoe_layer_config* cfg, const double* c_hat, const void* nccl_id128,
                          tamoe_layer** out);

/* Expert parallelism without NCCL (ranks may share a device: several ranks per GPU emulate a larger world).
 * Phase 1 creates this rank's layer and writes its TAMOE_EP_BLOB_BYTES blob (the CUDA IPC handle of its
 * workspace plus a fingerprint of the configuration / layout); the caller exchanges the blobs with any
 * transport (TCP store, MPI, gloo all-gather); phase 2 hands every rank's blob (world x 128 bytes, in rank
 * order) back and maps the peers.  A rank created with a different configuration is a validation error.
 * tamoe_layer_create_ep performs both phases over NCCL. */
#define TAMOE_EP_BLOB_BYTES 128
int tamoe_layer_create_ep_begin(const tamoe_layer_config* cfg, const double* c_hat, tamoe_layer** out,
                                void* blob_out);
int tamoe_layer_ep_connect(tamoe_layer* l, const void* blobs);
/* Off-rank payload bytes of the last step: out[4] = dispatch, expert-output return, dO, dX return. */
int tamoe_layer_a2a_bytes(tamoe_layer* l, long long* out4);
/* Host-side receive plan (CPU-testable): recv[P x E] rows per (source rank, local expert) -> the receive
 * segment of each local expert seg_start/seg_rows [E] (expert-major; inside it one 16-row padded block per
 * source rank, in rank order = the reference's (process, token) bucket order) and where each source's rows
 * for it start, src_off [P x E].  The device plan kernel computes the same from the all-gathered counts. */
int tamoe_ep_plan(int P, int E, const long long* recv, int* seg_start, int* seg_rows, long long* src_off);
int tamoe_layer_destroy(tamoe_layer* l);

/* ------------------------------------------------------------------ GPU-backed train() (§8(f) row 2)
 * train (trainer.cpp:183-452 / trainer.hpp:100-106): full-batch gradient descent on task MSE + aux_weight *
 * aux loss over P logical processes on this GPU (cfg.world_size = 1), per-process gate replicas, shared
 * experts, plain SGD in the reference's order on fp32 master weights.  kind: 0 balance, 1 topo, 2 compulsory
 * (not on the device path: validation error); cfg.aux_kind is derived from kind; topo switches to balance
 * after switch_step when has_switch.  x / y / wg / w1 / w2 are device bf16 in the layer layouts; the weights
 * are updated in place.  Report arrays are optional (null = not returned). */
typedef struct {
  int kind, steps;
  double lr;
  int has_switch, switch_step;
  int report_window;
  double bytes_per_element;
  const double* alpha_hat;   /* optional [P x P] profile for the per-step exchange estimate */
  const double* beta_hat;
  const int* intra_groups;   /* optional [P x P]: row i marks the devices of i's innermost group */
} tamoe_train_opts;

typedef struct {
  double* task_loss;         /* [steps] */
  double* aux_loss;          /* [steps] unweighted */
  double* comm_us;           /* [steps] bottleneck + size exchange (needs the profile) */
  double* dropped_rate;      /* [steps] */
  double* initial_dispatch;  /* [P x N] counts at step 0 */
  double* final_dispatch;    /* [P x N] averaged over the report window */
  double* tv_rows;           /* [P] TV(final row, c_hat row) (needs c_hat) */
  /* tv_initial_mean, tv_final_mean, col_balance_max_dev, min_expert_load, intra_share, final_task_loss,
   * final_aux_loss, final_comm_us, dropped_total_rate */
  double summary[9];
  double* comm_measured_us;  /* [steps] optional: the step's measured exchange in us (CUDA events, max over ranks):
                                counts exchange + dispatch phases under expert parallelism, the permute otherwise --
                                next to comm_us, the alpha-beta model of the same dispatch (comm_cost.cpp:24-55) */
} tamoe_train_report;

int tamoe_train(const tamoe_layer_config* cfg, const double* c_hat, const tamoe_train_opts* opts, const void* x,
                const void* y, void* wg, void* w1, void* w2, tamoe_train_report* report, void* stream);
/* train() in the reference's own precision (BASELINE C1): every step is tamoe_layer_step_f64 (fp64, linear
 * experts, the reference's summation order) followed by the fp64 SGD update (W -= lr * grad).  cfg supplies P, S,
 * d, d_out, N, k, cap_mode, capacity_factor, aux_weight, penalty_norm, temperature (f, act, need_dx ignored);
 * opts->kind 0 balance / 1 topo / 2 compulsory.  x [P*S x d], y [P*S x d_out], gates [P x d x N],
 * experts [N x d x d_out]: device fp64 in the reference's layouts, weights updated in place.  This is the
 * entry point of the drop-in train() replacement integration/tad_train_b200.cpp. */
int tamoe_train_f64(const tamoe_layer_config* cfg, const double* c_hat, const tamoe_train_opts* opts,
                    const double* x, const double* y, double* gates, double* experts, tamoe_train_report* report,
                    void* stream);
/* One layer step, stream-ordered, no host synchronisation.  A non-finite gate logit (the reference's
 * ValidationError, gate.cpp:16-17) cannot be reported by the call that enqueues the step: the device router
 * routes such a token to experts 0..k-1 with NaN gate values (indices stay in range, outputs and losses come
 * out NaN) and raises a flag that the next tamoe_layer_step (once the earlier step has completed) or
 * tamoe_layer_status returns as status 2. */
int tamoe_layer_step(tamoe_layer* l, const tamoe_layer_io* io, void* stream);
/* train() on an existing layer (any world size; trainer.cpp:183-452).  Under expert parallelism every rank calls it
 * with the same opts and c_hat [P_global x N], its own process' x / y, its gate replica wg and its E local experts
 * w1 / w2 (layer layouts, updated in place); each step the ranks exchange their losses, kept / dropped counts and
 * measured exchange time through the mapped workspaces, so the report (all P_global processes) is identical on
 * every rank.  opts->kind must match the layer's aux kind (topo -> balance switch allowed). */
int tamoe_layer_train(tamoe_layer* l, const double* c_hat, const tamoe_train_opts* opts, const void* x, const void* y,
                      void* wg, void* w1, void* w2, tamoe_train_report* report, void* stream);
/* Waits for the last step; status 2 ("non-finite gate logit") if it saw a non-finite logit (reported once). */
int tamoe_layer_status(tamoe_layer* l);
int tamoe_layer_read(tamoe_layer* l, int what, void* dst, long long bytes, void* stream);
int tamoe_layer_n_pad(int N);
/* Kernel launches of libtamoe per step (memsets excluded). */
int tamoe_layer_launches_per_step(tamoe_layer* l);
/* Per-launch CUDA-event timing of the step on its stream (enable != 0 turns it on and resets totals).
 * tamoe_layer_timing reads accumulated milliseconds per launch slot: names[i] (static strings), ms[i];
 * returns the slot count through *n and the number of timed steps through *steps. */
int tamoe_layer_enable_timing(tamoe_layer* l, int enable);
int tamoe_layer_timing(tamoe_layer* l, const char** names, double* ms, int cap, int* n, int* steps);

#ifdef __cplusplus
}
#endif

#endif /* TAMOE_H_ */
