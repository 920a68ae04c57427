// Drop-in replacement for the reference's train() (proj/core/src/trainer.cpp:183-457), backed by the B200 library.
//
// The reference inlines its MoE layer in train(): per step gate_forward, topk_route (+ apply_compulsory_quota),
// the linear experts, combine, task MSE, the backward and the SGD update, all fp64 on one host thread.  Here the
// whole step runs on the GPU through tamoe_train_f64 (include/tamoe.h): tamoe_layer_step_f64 in the reference's
// summation order without FMA, then the fp64 SGD update; the report bookkeeping (losses, comm estimate, dropped
// rate, window dispatch, TV, balance, intra share) is restated in the library from the per-step device counters.
//
// Everything train() does before its step loop is host-side set-up and stays here, restated against the
// reference's own headers: the argument checks (trainer.cpp:186-192) and the seeded weight initialisation when
// the config carries no explicit start (trainer.cpp:207-225: gate W_i = 0.01 N(0,1) from
// derive_seed(seed, 2000 + i), expert U_e = N(0,1) / sqrt(d) from derive_seed(seed, 3000 + e), row-major).
//
// Built by oracle/ref.mk (`make -f oracle/ref.mk suite_b200_train`): the reference's own unit suite linked
// against the reference objects with train() renamed away in trainer.o, this file, and the gate.cpp shim.
#include <cuda_runtime.h>

#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "tadispatch/errors.hpp"
#include "tadispatch/rng.hpp"
#include "tadispatch/trainer.hpp"
#include "tamoe.h"

namespace tad {
namespace {

void check(int status) {
  if (status == TAMOE_OK) return;
  if (status == TAMOE_ERR_VALIDATION) throw ValidationError(tamoe_last_error());
  throw std::runtime_error(tamoe_last_error());
}

void cuda(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

struct DeviceArray {
  double* p = nullptr;
  explicit DeviceArray(const std::vector<double>& host) {
    cuda(cudaMalloc(&p, sizeof(double) * (host.empty() ? 1 : host.size())));
    if (!host.empty()) cuda(cudaMemcpy(p, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice));
  }
  ~DeviceArray() { cudaFree(p); }
  DeviceArray(const DeviceArray&) = delete;
  DeviceArray& operator=(const DeviceArray&) = delete;
};

void append(std::vector<double>& dst, const Matrix& m) {
  dst.insert(dst.end(), m.data().begin(), m.data().end());
}

Matrix to_matrix(const std::vector<double>& v, int rows, int cols) {
  Matrix m(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) m.at(i, j) = v[static_cast<size_t>(i) * cols + j];
  return m;
}

}  // namespace

TrainReport train(const TrainConfig& config, const SyntheticTask& task, LossKind kind, const Matrix* c_hat) {
  const ModelDims& dims = config.dims;
  const int P = dims.P, N = dims.N, S = dims.S, d = dims.d, d_out = dims.d_out;
  if (N % P != 0) throw ValidationError("N must be divisible by P");
  if (static_cast<int>(task.batch_x.size()) != P)
    throw ValidationError("task was generated for a different process count");
  if (kind != LossKind::balance && c_hat == nullptr)
    throw ValidationError("topo and compulsory losses require a target pattern");
  if (c_hat && (c_hat->rows() != P || c_hat->cols() != N)) throw ValidationError("target pattern must be P x N");

  // initial weights: the config's explicit start, else the seeded init
  std::vector<double> gates, experts;
  if (config.init_gates.empty()) {
    for (int i = 0; i < P; ++i) {
      Rng rng(derive_seed(config.seed, 2000 + static_cast<uint64_t>(i)));
      for (long long j = 0; j < static_cast<long long>(d) * N; ++j) gates.push_back(0.01 * rng.normal());
    }
  } else {
    for (const Matrix& m : config.init_gates) append(gates, m);
  }
  if (config.init_experts.empty()) {
    const double scale = 1.0 / std::sqrt(static_cast<double>(d));
    for (int e = 0; e < N; ++e) {
      Rng rng(derive_seed(config.seed, 3000 + static_cast<uint64_t>(e)));
      for (long long j = 0; j < static_cast<long long>(d) * d_out; ++j) experts.push_back(scale * rng.normal());
    }
  } else {
    for (const Matrix& m : config.init_experts) append(experts, m);
  }
  if (static_cast<long long>(gates.size()) != static_cast<long long>(P) * d * N ||
      static_cast<long long>(experts.size()) != static_cast<long long>(N) * d * d_out)
    throw ValidationError("initial weights have the wrong process or expert count");

  std::vector<double> xs, ys, ch, alpha, beta;
  for (int i = 0; i < P; ++i) {
    append(xs, task.batch_x[static_cast<size_t>(i)]);
    append(ys, task.batch_y[static_cast<size_t>(i)]);
  }
  if (c_hat) append(ch, *c_hat);
  const bool has_profile = config.alpha_hat.rows() == P && config.beta_hat.rows() == P;
  if (has_profile) {
    append(alpha, config.alpha_hat);
    append(beta, config.beta_hat);
  }
  std::vector<int> intra;
  if (!config.intra_groups.empty()) {
    intra.assign(static_cast<size_t>(P) * P, 0);
    for (int i = 0; i < P; ++i)
      for (int dev : config.intra_groups[static_cast<size_t>(i)]) intra[static_cast<size_t>(i) * P + dev] = 1;
  }

  DeviceArray dx(xs), dy(ys), dg(gates), de(experts);
  tamoe_layer_config cfg{};
  cfg.P = P;
  cfg.S = S;
  cfg.d = d;
  cfg.d_out = d_out;
  cfg.N = N;
  cfg.k = dims.k;
  cfg.cap_mode = static_cast<int>(config.capacity.mode);
  cfg.capacity_factor = config.capacity.capacity_factor;
  cfg.aux_weight = config.aux_weight;
  cfg.penalty_norm = static_cast<int>(config.norm);
  cfg.temperature = config.temperature;
  cfg.world_size = 1;
  tamoe_train_opts opts{};
  opts.kind = static_cast<int>(kind);
  opts.steps = config.steps;
  opts.lr = config.lr;
  opts.has_switch = config.switch_step.has_value() ? 1 : 0;
  opts.switch_step = config.switch_step.value_or(0);
  opts.report_window = config.report_window;
  opts.bytes_per_element = dims.bytes_per_element;
  opts.alpha_hat = has_profile ? alpha.data() : nullptr;
  opts.beta_hat = has_profile ? beta.data() : nullptr;
  opts.intra_groups = intra.empty() ? nullptr : intra.data();

  const int steps = config.steps > 0 ? config.steps : 0;
  std::vector<double> task_loss(steps), aux_loss(steps), comm(steps), dropped(steps), d0(static_cast<size_t>(P) * N),
      d1(static_cast<size_t>(P) * N), tv(static_cast<size_t>(P));
  tamoe_train_report rep{};
  rep.task_loss = task_loss.data();
  rep.aux_loss = aux_loss.data();
  rep.comm_us = comm.data();
  rep.dropped_rate = dropped.data();
  rep.initial_dispatch = d0.data();
  rep.final_dispatch = d1.data();
  rep.tv_rows = tv.data();
  check(tamoe_train_f64(&cfg, c_hat ? ch.data() : nullptr, &opts, dx.p, dy.p, dg.p, de.p, &rep, nullptr));

  TrainReport report;
  report.loss = kind;
  report.seed = config.seed;
  report.task_loss = task_loss;
  report.aux_loss = aux_loss;
  report.comm_us = comm;
  report.dropped_rate = dropped;
  report.initial_dispatch = to_matrix(d0, P, N);
  report.final_dispatch = to_matrix(d1, P, N);
  if (steps == 0) return report;
  if (c_hat) report.tv_rows = tv;
  report.tv_initial_mean = rep.summary[0];
  report.tv_final_mean = rep.summary[1];
  report.col_balance_max_dev = rep.summary[2];
  report.min_expert_load = rep.summary[3];
  report.intra_share = rep.summary[4];
  report.final_task_loss = rep.summary[5];
  report.final_aux_loss = rep.summary[6];
  report.final_comm_us = rep.summary[7];
  report.dropped_total_rate = rep.summary[8];
  return report;
}

}  // namespace tad
