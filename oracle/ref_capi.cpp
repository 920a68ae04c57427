// TEST INFRASTRUCTURE ONLY -- C wrapper around the reference library compiled
// from its own, unmodified sources under /root/reference/proj/core/src (see
// oracle/ref.mk).  Output: oracle/_ref/libtadref.so.  Used to pin the C
// restatement (oracle/tamoe_oracle.c), to generate tests/golden fixtures and as
// the CPU baseline of bench.py (cpu_baseline.kind = "reference").
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "tadispatch/comm_cost.hpp"
#include "tadispatch/errors.hpp"
#include "tadispatch/gate.hpp"
#include "tadispatch/profile.hpp"
#include "tadispatch/profile_io.hpp"
#include "tadispatch/topology.hpp"
#include "tadispatch/rng.hpp"
#include "tadispatch/solver.hpp"
#include "tadispatch/trainer.hpp"

using namespace tad;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

Matrix to_matrix(const double* p, int r, int c) {
  Matrix m(r, c);
  if (r * c) std::memcpy(m.data().data(), p, sizeof(double) * r * c);
  return m;
}
void from_matrix(const Matrix& m, double* out) {
  if (!m.data().empty()) std::memcpy(out, m.data().data(), sizeof(double) * m.data().size());
}
CapacityMode mode_of(int m) {
  switch (m) {
    case 1: return CapacityMode::global;
    case 2: return CapacityMode::local;
    case 3: return CapacityMode::local_proportional;
    default: return CapacityMode::none;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// tad::Rng stream: n draws of scale * normal() (test_gate.cpp:14-18 random_matrix).
void ref_rng_normal(unsigned long long seed, int n, double scale, double* out) {
  Rng rng(seed);
  for (int i = 0; i < n; ++i) out[i] = scale * rng.normal();
}
void ref_rng_uniform(unsigned long long seed, int n, double lo, double hi, double* out) {
  Rng rng(seed);
  for (int i = 0; i < n; ++i) out[i] = rng.uniform(lo, hi);
}
unsigned long long ref_derive_seed(unsigned long long seed, unsigned long long stream) {
  return derive_seed(seed, stream);
}

int ref_softmax_rows(const double* logits, int S, int N, double* probs) {
  return guard([&] { from_matrix(softmax_rows(to_matrix(logits, S, N)), probs); });
}

int ref_gate_forward(const double* x, const double* W, int S, int d, int N, double* probs) {
  return guard([&] { from_matrix(gate_forward(to_matrix(x, S, d), to_matrix(W, d, N)), probs); });
}

void ref_largest_remainder_round(const double* v, int n, long long target, long long* out) {
  auto r = largest_remainder_round(std::span<const double>(v, static_cast<size_t>(n)), target);
  for (int i = 0; i < n; ++i) out[i] = r[static_cast<size_t>(i)];
}

int ref_topk_route(const double* probs, int P, int S, int N, int k, int mode, double cf, const double* c_hat,
                   int* expert, double* gate, double* score, unsigned char* kept, long long* counts,
                   long long* dropped, double* mean_probs) {
  return guard([&] {
    std::vector<Matrix> pp;
    for (int i = 0; i < P; ++i) pp.push_back(to_matrix(probs + static_cast<size_t>(i) * S * N, S, N));
    Matrix ch;
    if (c_hat) ch = to_matrix(c_hat, P, N);
    auto res = topk_route(pp, k, CapacityPolicy{mode_of(mode), cf}, c_hat ? &ch : nullptr);
    for (int i = 0; i < P; ++i) {
      const auto& r = res[static_cast<size_t>(i)];
      for (int s = 0; s < S; ++s)
        for (int slot = 0; slot < k; ++slot) {
          const size_t a = (static_cast<size_t>(i) * S + s) * k + slot;
          const auto& as = r.assignments[static_cast<size_t>(s)][static_cast<size_t>(slot)];
          expert[a] = as.expert;
          gate[a] = as.gate_value;
          score[a] = as.score;
          kept[a] = as.kept ? 1 : 0;
        }
      for (int e = 0; e < N; ++e) {
        counts[static_cast<size_t>(i) * N + e] = r.counts[static_cast<size_t>(e)];
        dropped[static_cast<size_t>(i) * N + e] = r.dropped[static_cast<size_t>(e)];
        mean_probs[static_cast<size_t>(i) * N + e] = r.mean_probs[static_cast<size_t>(e)];
      }
    }
  });
}

int ref_penalty_weights(const double* c_hat_row, int n, int norm, double temperature, double* p) {
  return guard([&] {
    auto r = penalty_weights(std::span<const double>(c_hat_row, static_cast<size_t>(n)),
                             norm == 0 ? PenaltyNorm::sum_norm : PenaltyNorm::softmax, temperature);
    std::memcpy(p, r.data(), sizeof(double) * r.size());
  });
}

static RoutingResult make_result(const long long* counts, const double* mean_probs, int N) {
  RoutingResult r;
  r.counts.assign(counts, counts + N);
  r.dropped.assign(static_cast<size_t>(N), 0);
  r.mean_probs.assign(mean_probs, mean_probs + N);
  return r;
}

double ref_loss_balance(const long long* counts, const double* mean_probs, int N, int S) {
  return loss_balance(make_result(counts, mean_probs, N), S);
}

int ref_loss_topo(const long long* counts, const double* mean_probs, const double* p, int N, int P, int S,
                  double* out) {
  return guard([&] {
    *out = loss_topo(make_result(counts, mean_probs, N), std::span<const double>(p, static_cast<size_t>(N)), N, P, S);
  });
}

int ref_grad_loss_topo(const double* x, const double* probs, const long long* counts, const double* mean_probs,
                       const double* p, int S, int d, int N, int P, double* grad) {
  return guard([&] {
    from_matrix(grad_loss_topo(to_matrix(x, S, d), to_matrix(probs, S, N), make_result(counts, mean_probs, N),
                               std::span<const double>(p, static_cast<size_t>(N)), N, P, S),
                grad);
  });
}

int ref_grad_loss_balance(const double* x, const double* probs, const long long* counts, const double* mean_probs,
                          int S, int d, int N, double* grad) {
  return guard([&] {
    from_matrix(grad_loss_balance(to_matrix(x, S, d), to_matrix(probs, S, N), make_result(counts, mean_probs, N), S),
                grad);
  });
}

int ref_target_closed_form(const double* beta, int P, int N, int k, int S, double* c_hat) {
  return guard([&] {
    DispatchConfig dc{k, S, N, P, 1.0, 4.0};
    from_matrix(target_closed_form(to_matrix(beta, P, P), dc).dispatch.c, c_hat);
  });
}

// gen_synthetic (trainer.cpp:57-104): per-process batches x[P][S][d], y[P][S][d_out].
int ref_gen_synthetic(unsigned long long seed, int P, int S, int d, int d_out, int N, int k, int clusters,
                      double separation, double within_std, double noise_std, double map_spread, double* x,
                      double* y, double* cluster_means, double* true_maps) {
  return guard([&] {
    ModelDims dims{d, d_out, N, P, k, S, 4.0};
    TaskConfig task{clusters, separation, within_std, noise_std, map_spread};
    SyntheticTask t = gen_synthetic(seed, dims, task);
    for (int i = 0; i < P; ++i) {
      from_matrix(t.batch_x[static_cast<size_t>(i)], x + static_cast<size_t>(i) * S * d);
      from_matrix(t.batch_y[static_cast<size_t>(i)], y + static_cast<size_t>(i) * S * d_out);
    }
    if (cluster_means) from_matrix(t.cluster_means, cluster_means);
    if (true_maps)
      for (int c = 0; c < clusters; ++c)
        from_matrix(t.true_maps[static_cast<size_t>(c)], true_maps + static_cast<size_t>(c) * d * d_out);
  });
}

// train() (trainer.cpp:183-457) on caller-provided batches and initial weights.
// kind: 0 balance, 1 topo, 2 compulsory.  switch_step < -1000000 disables it.
// Outputs: task_loss/aux_loss/dropped_rate [steps], initial/final dispatch [P x N].
int ref_train(int P, int S, int d, int d_out, int N, int k, const double* x, const double* y, const double* gates,
              const double* experts, int kind, int cap_mode, double cf, const double* c_hat, int norm,
              double temperature, double lr, int steps, double aux_weight, int switch_step, double* task_loss,
              double* aux_loss, double* dropped_rate, double* initial_dispatch, double* final_dispatch,
              double* seconds) {
  return guard([&] {
    TrainConfig cfg;
    cfg.dims = ModelDims{d, d_out, N, P, k, S, 4.0};
    cfg.lr = lr;
    cfg.steps = steps;
    cfg.aux_weight = aux_weight;
    cfg.norm = norm == 0 ? PenaltyNorm::sum_norm : PenaltyNorm::softmax;
    cfg.temperature = temperature;
    cfg.capacity = CapacityPolicy{mode_of(cap_mode), cf};
    if (switch_step > -1000000) cfg.switch_step = switch_step;
    for (int i = 0; i < P; ++i) cfg.init_gates.push_back(to_matrix(gates + static_cast<size_t>(i) * d * N, d, N));
    for (int e = 0; e < N; ++e)
      cfg.init_experts.push_back(to_matrix(experts + static_cast<size_t>(e) * d * d_out, d, d_out));
    SyntheticTask task;
    for (int i = 0; i < P; ++i) {
      task.batch_x.push_back(to_matrix(x + static_cast<size_t>(i) * S * d, S, d));
      task.batch_y.push_back(to_matrix(y + static_cast<size_t>(i) * S * d_out, S, d_out));
    }
    Matrix ch;
    if (c_hat) ch = to_matrix(c_hat, P, N);
    const LossKind lk = kind == 1 ? LossKind::topo : (kind == 2 ? LossKind::compulsory : LossKind::balance);
    const auto t0 = std::chrono::steady_clock::now();
    TrainReport rep = train(cfg, task, lk, c_hat ? &ch : nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    for (int s = 0; s < steps; ++s) {
      if (task_loss) task_loss[s] = rep.task_loss[static_cast<size_t>(s)];
      if (aux_loss) aux_loss[s] = rep.aux_loss[static_cast<size_t>(s)];
      if (dropped_rate) dropped_rate[s] = rep.dropped_rate[static_cast<size_t>(s)];
    }
    if (initial_dispatch) from_matrix(rep.initial_dispatch, initial_dispatch);
    if (final_dispatch) from_matrix(rep.final_dispatch, final_dispatch);
  });
}

// ---- measured-topology pipeline (comm_cost.cpp, profile.cpp, topology.cpp)
static Topology tree_from_levels(const int* levels, int n_levels) {
  std::string t = "[";
  for (int i = 0; i < n_levels; ++i) t += (i ? "," : "") + std::to_string(levels[i]);
  return parse_topology(t + "]");
}

int ref_fit_profile(const int* src, const int* dst, const double* mb, const double* us, int n, int P, double* alpha,
                    double* beta) {
  return guard([&] {
    std::vector<TransferSample> smp;
    for (int i = 0; i < n; ++i) smp.push_back({src[i], dst[i], mb[i], us[i]});
    FittedProfile f = fit_profile(smp, P);
    std::memcpy(alpha, f.alpha.data().data(), sizeof(double) * P * P);
    std::memcpy(beta, f.beta.data().data(), sizeof(double) * P * P);
  });
}

int ref_fill_partial_profile(const double* alpha, const double* beta, int P, const int* levels, int n_levels,
                             double floor, double* alpha_out, double* beta_out) {
  return guard([&] {
    Topology topo;
    if (n_levels > 0) topo = tree_from_levels(levels, n_levels);
    LinkProfile lp = fill_partial_profile(to_matrix(alpha, P, P), to_matrix(beta, P, P),
                                          n_levels > 0 ? &topo : nullptr, floor);
    std::memcpy(alpha_out, lp.alpha.data().data(), sizeof(double) * P * P);
    std::memcpy(beta_out, lp.beta.data().data(), sizeof(double) * P * P);
  });
}

int ref_smooth_profile(const int* levels, int n_levels, const double* alpha, const double* beta, int P, double floor,
                       double* alpha_hat, double* beta_hat) {
  return guard([&] {
    Topology topo = tree_from_levels(levels, n_levels);
    LinkProfile raw;
    raw.alpha = to_matrix(alpha, P, P);
    raw.beta = to_matrix(beta, P, P);
    raw.self_beta_floor = floor;
    HierarchicalProfile h = smooth_profile(topo, raw);
    std::memcpy(alpha_hat, h.alpha_hat.data().data(), sizeof(double) * P * P);
    std::memcpy(beta_hat, h.beta_hat.data().data(), sizeof(double) * P * P);
  });
}

int ref_device_groups(const int* levels, int n_levels, int device, int* group_of /* [P] */) {
  return guard([&] {
    Topology topo = tree_from_levels(levels, n_levels);
    auto g = device_groups(topo, device);
    for (size_t l = 0; l < g.size(); ++l)
      for (int j : g[l]) group_of[j] = static_cast<int>(l);
  });
}

int ref_exchange_cost(const double* alpha, const double* beta, const double* c, int P, int N, int d, int b,
                      int rounds, double* pair_cost, double* summary) {
  return guard([&] {
    DispatchMatrix dm;
    dm.config.P = P;
    dm.config.N = N;
    dm.config.d = d;
    dm.config.b = b;
    dm.config.k = 1;
    dm.config.S = 1;
    dm.c = to_matrix(c, P, N);
    CostReport r = exchange_cost(to_matrix(alpha, P, P), to_matrix(beta, P, P), dm, rounds);
    std::memcpy(pair_cost, r.pair_cost_us.data().data(), sizeof(double) * P * P);
    summary[0] = r.bottleneck_us;
    summary[1] = r.total_bytes;
    summary[2] = r.size_exchange_us;
    summary[3] = r.total_estimate_us;
  });
}

}  // extern "C"
