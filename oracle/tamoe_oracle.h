/*
 * TEST INFRASTRUCTURE ONLY -- the parity oracle for the TA-MoE hot path.
 *
 * A plain-C, fp64 restatement of the reference's CPU algorithm
 * (/root/reference/proj/core/src/gate.cpp, trainer.cpp:243-482,
 * solver.cpp:28-52, dispatch.cpp:21-26).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker.  The
 * product (libtamoe.so) never links or calls it.
 *
 * Parity pinning: tests/test_oracle_ref.py checks this restatement against the
 * reference compiled from its own sources (oracle/_ref, built by oracle/ref.mk)
 * and against the committed golden fixtures under tests/golden/.  The linear
 * expert path is bit-identical to the reference (same loop order, same
 * association); the FFN expert (d -> f -> d_out) and dX are extensions the
 * reference does not have ("parity unpinned" for those two, FD-checked instead).
 *
 * Layout: row-major, flat arrays.  Status: 0 ok, 2 validation error.
 */
#ifndef TAMOE_ORACLE_H_
#define TAMOE_ORACLE_H_

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_CAP_NONE = 0, ORC_CAP_GLOBAL = 1, ORC_CAP_LOCAL = 2, ORC_CAP_PROPORTIONAL = 3 };
enum { ORC_AUX_BALANCE = 0, ORC_AUX_TOPO = 1 };
enum { ORC_ACT_NONE = 0, ORC_ACT_GELU = 1, ORC_ACT_RELU = 2 };

const char* orc_last_error(void);

/* gate.cpp:12-28 */
int orc_softmax_rows(const double* logits, int S, int N, double* probs);
/* matrix.hpp:82-93 (C = A B, i-k-j, zero a_ik skipped) */
void orc_matmul(const double* a, const double* b, int n, int kdim, int m, double* c);
/* gate.cpp:30-32 */
int orc_gate_forward(const double* x, const double* W, int S, int d, int N, double* probs);
/* gate.cpp:52-78 */
void orc_largest_remainder_round(const double* values, int n, long long target, long long* out);
/* gate.cpp:91-202 for P processes; per-process arrays are concatenated (process-major). */
int orc_topk_route(const double* probs, int P, int S, int N, int k, int mode, double cf, const double* c_hat,
                   int* expert, double* gate, double* score, unsigned char* kept, long long* counts,
                   long long* dropped, double* mean_probs);
/* gate.cpp:209-214 */
double orc_loss_balance(const long long* counts, const double* mean_probs, int N, int S);
/* gate.cpp:222-246 */
int orc_penalty_weights(const double* c_hat_row, int n, int norm, double temperature, double* p);
/* gate.cpp:248-255 */
double orc_loss_topo(const long long* counts, const double* mean_probs, const double* penalty, int N, int P, int S);
/* gate.cpp:257-287: coefficient vectors, then dW = x^T [p * (coeff - <coeff,p>)] */
void orc_balance_coefficients(const long long* counts, int N, int S, double* coeff);
void orc_topo_coefficients(const long long* counts, const double* penalty, int N, int P, int S, double* coeff);
void orc_grad_aux_loss(const double* x, const double* probs, const double* coeff, int S, int d, int N, double* grad);
/* solver.cpp:28-52 */
int orc_target_closed_form(const double* beta_hat, int P, int N, int k, int S, double* c_hat);
/* trainer.cpp:121-169 (top-1 compulsory quota ablation), in place on one process' routing */
int orc_apply_compulsory_quota(const double* probs, const double* c_hat_row, int S, int N, int* expert,
                               double* gate, double* score, unsigned char* kept, long long* counts,
                               long long* dropped);

/* One MoE-layer training step (trainer.cpp:371-482) over all P processes.
 * Linear experts (f == 0): U[N][d][d_out], exactly the reference.  FFN experts (f > 0):
 * W1[N][d][f], W2[N][f][d_out], out = act(x W1) W2 (extension).
 * penalties[P][N] used when aux_kind == ORC_AUX_TOPO.
 * Outputs (all optional except losses): probs[P*S*N], routing arrays [P*S*k], counts/dropped/mean_probs[P*N],
 * y_hat[P*S*d_out], gate_grads[P][d][N], expert grads with the weights' shapes, dx[P*S*d] (extension). */
typedef struct {
  int P, S, d, d_out, N, k, f, act;
  int cap_mode;
  double cf;
  int aux_kind;
  double aux_weight;
  const double* c_hat;      /* P x N, required for proportional capacity */
  const double* penalties;  /* P x N, required for topo aux */
} orc_layer_cfg;

typedef struct {
  double* probs;
  int* expert;
  double* gate;
  double* score;
  unsigned char* kept;
  long long* counts;
  long long* dropped;
  double* mean_probs;
  double* y_hat;
  double task_loss;
  double aux_loss;
  double* gate_grads;
  double* grad_u;   /* linear: N*d*d_out */
  double* grad_w1;  /* ffn: N*d*f */
  double* grad_w2;  /* ffn: N*f*d_out */
  double* dx;
} orc_layer_out;

int orc_layer_step(const orc_layer_cfg* cfg, const double* x, const double* y, const double* gates,
                   const double* U, const double* W1, const double* W2, orc_layer_out* out);

#ifdef __cplusplus
}
#endif
#endif
