// GPU-backed train(): full-batch gradient descent of the TA-MoE layer on task MSE +
// aux_weight * auxiliary loss, per-process gate replicas, shared experts, fp32 master weights, and the
// reference's TrainReport (trainer.hpp:75-99, trainer.cpp:183-452) computed from the device counters.
#pragma once
#include <climits>
#include <vector>

#include "layer.hpp"

namespace tamoe {

struct TrainOptions {
  int kind = 0;                  // 0 balance, 1 topo, 2 compulsory (LossKind)
  int steps = 1;
  double lr = 0.05;
  int switch_step = INT_MIN;     // topo -> balance after this step (INT_MIN: never)
  int report_window = 100;
  double bytes_per_element = 4.0;
  const double* alpha_hat = nullptr;  // [P x P] optional profile for the per-step comm estimate
  const double* beta_hat = nullptr;
  const int* intra_groups = nullptr;  // [P x P] optional: row i marks the devices of i's innermost group
};

struct TrainReport {
  std::vector<double> task_loss, aux_loss, comm_us, dropped_rate;  // per step
  std::vector<double> comm_measured_us;  // per step: the measured exchange (CUDA events; max over ranks)
  std::vector<double> initial_dispatch, final_dispatch;           // [P x N]
  std::vector<double> tv_rows;                                    // [P] (with c_hat)
  double tv_initial_mean = 0, tv_final_mean = 0, col_balance_max_dev = 0, min_expert_load = 0;
  double intra_share = 0, final_task_loss = 0, final_aux_loss = 0, final_comm_us = 0, dropped_total_rate = 0;
};

// x [P*S x d], y [P*S x d_out] (bf16, device); wg / w1 / w2 (bf16, device, the layer's layouts) are the
// initial weights on entry and the trained weights on return.  cfg.aux_kind is derived from opts.kind.
TrainReport train_layer(LayerConfig cfg, const double* c_hat, const TrainOptions& opts, const __nv_bfloat16* x,
                        const __nv_bfloat16* y, __nv_bfloat16* wg, __nv_bfloat16* w1, __nv_bfloat16* w2,
                        cudaStream_t s);

// The loop on an existing layer -- any world size: under expert parallelism every rank passes its own process'
// x / y, its gate replica wg and its E = N / world local experts; the report covers all world * P processes and
// is identical on every rank (losses, counts and the measured exchange are gathered each step).
TrainReport train_on_layer(Layer& layer, const double* c_hat, const TrainOptions& opts, const __nv_bfloat16* x,
                           const __nv_bfloat16* y, __nv_bfloat16* wg, __nv_bfloat16* w1, __nv_bfloat16* w2,
                           cudaStream_t s);

// The same loop in the reference's own precision (BASELINE C1): fp64 device step (layer_step_f64, linear experts)
// and fp64 SGD.  x [P*S x d], y [P*S x d_out], gates [P x d x N], experts [N x d x d_out]: device fp64 in the
// reference's layouts; gates / experts are the initial weights on entry and the trained weights on return.
TrainReport train_f64(int P, int S, int d, int d_out, int N, int k, int cap_mode, double cf, double aux_weight,
                      int norm, double temperature, const double* c_hat, const TrainOptions& opts, const double* x,
                      const double* y, double* gates, double* experts, cudaStream_t s);

double tv_distance(const double* a, const double* b, int n);  // trainer.cpp:88-96

}  // namespace tamoe
