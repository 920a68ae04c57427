// Reference-precision MoE layer step (fp64, linear experts) -- BASELINE config 1 on the device.
//
// The reference layer is fp64 end to end with a linear expert (trainer.cpp:246-356).  The bf16 tcgen05 layer
// (layer.cpp) is the throughput path; this step reproduces the reference's arithmetic for the parity
// configuration: every per-element sum runs in the reference's order with separately rounded products
// (no FMA), so expert outputs, dL/dg, expert / gate gradients and the aux terms are bit-identical to the
// reference whenever the softmax is (CUDA's exp is <= 1 ulp from glibc's); the task loss is summed per token
// first (the reference uses one running sum), which moves it by a few ulp.
#pragma once
#include <cuda_runtime.h>

#include "layer.hpp"

namespace tamoe {

struct F64StepArgs {
  int d = 0, d_out = 0;
  const double* x = nullptr;        // device [P*S x d]
  const double* y = nullptr;        // device [P*S x d_out]
  const double* gates = nullptr;    // device [P x d x N]   (GateState::W per process, trainer.cpp:207-216)
  const double* experts = nullptr;  // device [N x d x d_out] (linear experts U_e, trainer.cpp:219-223)
  const double* penalty = nullptr;  // host [P x N] (topo loss only)
  const double* c_hat = nullptr;    // host [P x N] (compulsory quotas only)
  int aux_kind = 0;                 // 0 balance, 1 topo, 2 compulsory (quota routing, balance loss)
  double aux_weight = 1.0;
  int cap_mode = 0;
  const long long* caps = nullptr;  // host [P x N] (tamoe_capacity_caps)
  double* probs = nullptr;          // device [P*S x N] out (optional)
  double* gate_grads = nullptr;     // device [P x d x N] out
  double* expert_grads = nullptr;   // device [N x d x d_out] out
  double* y_hat = nullptr;          // device [P*S x d_out] out (optional)
  double* losses = nullptr;         // host [2] out: task loss, aux loss (trainer.cpp:359-360)
};

// Gate (per-process fp64 gate_forward) -> topk_route on the router workspace -> linear experts -> combine ->
// MSE -> backward (dL/dg, top-k renormalisation Jacobian, aux coefficients, softmax backward, x^T dz).
// Synchronises `s` (validation of the logits, the losses returned to the host).
void layer_step_f64(RouteWorkspace& rw, const F64StepArgs& a, cudaStream_t s);

}  // namespace tamoe
