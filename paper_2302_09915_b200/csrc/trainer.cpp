// GPU-backed train(): the step loop of trainer.cpp:247-417 around Layer::step, with the report bookkeeping
// of trainer.cpp:227-452 restated on the host from the per-step device counters (losses, kept / dropped
// counts).  The SGD update runs on fp32 master weights (sgd.cu); the layer reads their bf16 copies.
#include "trainer.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.hpp"
#include "host_topology.hpp"
#include "layer_f64.hpp"
#include "sgd.hpp"

namespace tamoe {

double tv_distance(const double* a, const double* b, int n) {
  double sa = 0.0, sb = 0.0;
  for (int e = 0; e < n; ++e) sa += a[e];
  for (int e = 0; e < n; ++e) sb += b[e];
  if (!(sa > 0.0) || !(sb > 0.0)) return 0.0;
  double tv = 0.0;
  for (int e = 0; e < n; ++e) tv += std::abs(a[e] / sa - b[e] / sb);
  return 0.5 * tv;
}

namespace {

template <class T>
T* dalloc(long long n) {
  T* p = nullptr;
  TAMOE_CUDA(cudaMalloc(&p, sizeof(T) * static_cast<size_t>(n > 0 ? n : 1)));
  TAMOE_CUDA(cudaMemset(p, 0, sizeof(T) * static_cast<size_t>(n > 0 ? n : 1)));
  return p;
}

struct DevBuf {
  std::vector<void*> ptrs;
  template <class T>
  T* get(long long n) {
    T* p = dalloc<T>(n);
    ptrs.push_back(p);
    return p;
  }
  ~DevBuf() {
    for (void* p : ptrs) cudaFree(p);
  }
};

}  // namespace

namespace {

// The bookkeeping of train() (trainer.cpp:227-452) around a device step: `step(i, losses, counts, dropped)` runs
// step i (forward, backward, the synchronized SGD update) and returns its task / aux loss and the per-(process,
// expert) kept / dropped counts; everything the report derives from them is restated here on the host.
template <class Step>
TrainReport run_train(int P, int S, int N, int k, int d, int cap_mode, double aux_weight, const double* c_hat,
                      const TrainOptions& o, Step&& step_fn) {
  const int E = N / P;
  const bool has_profile = o.alpha_hat != nullptr && o.beta_hat != nullptr;
  const int rounds = (cap_mode == 1 || cap_mode == 3) ? 1 : 0;  // global / proportional: size round
  TrainReport rep;
  const int window = std::max(1, std::min(o.report_window, std::max(o.steps, 1)));
  const int window_start = std::max(0, o.steps - window);
  std::vector<double> dsum(static_cast<size_t>(P) * N, 0.0);
  long long win_steps = 0, dropped_total = 0;
  double win_task = 0, win_aux = 0, win_comm = 0, intra_num = 0, intra_den = 0;
  std::vector<int> counts_i(static_cast<size_t>(P) * N), dropped_i(static_cast<size_t>(P) * N);
  std::vector<double> counts(static_cast<size_t>(P) * N);
  double losses[2];

  for (int step = 0; step < o.steps; ++step) {
    double measured = 0.0;
    step_fn(step, losses, counts_i.data(), dropped_i.data(), &measured);
    rep.comm_measured_us.push_back(measured);
    const double task = losses[0], aux = losses[1];
    if (!std::isfinite(task + aux_weight * aux))
      throw std::runtime_error("training diverged at step " + std::to_string(step) + " (task=" +
                               std::to_string(task) + ", aux=" + std::to_string(aux) + "); lower the learning rate");
    long long dropped_step = 0;
    for (size_t i = 0; i < counts.size(); ++i) {
      counts[i] = counts_i[i];
      dropped_step += dropped_i[i];
    }
    dropped_total += dropped_step;
    double comm = 0.0;
    if (has_profile) {
      // DispatchConfig{k, S, N, P, d, b}: payload of d * bytes_per_element per token (trainer.cpp:239)
      const double mb_per_token = d * o.bytes_per_element / 1e6;
      const std::vector<double> pay = device_payload_tokens(counts.data(), P, N);
      double bott = 0.0, max_alpha = 0.0;
      for (int i = 0; i < P * P; ++i) {
        bott = std::max(bott, o.alpha_hat[i] + o.beta_hat[i] * (pay[static_cast<size_t>(i)] * mb_per_token));
        max_alpha = std::max(max_alpha, o.alpha_hat[i]);
      }
      comm = bott + rounds * max_alpha;
    }
    rep.task_loss.push_back(task);
    rep.aux_loss.push_back(aux);
    rep.comm_us.push_back(comm);
    rep.dropped_rate.push_back(static_cast<double>(dropped_step) / (static_cast<double>(k) * S * P));
    if (step == 0) rep.initial_dispatch = counts;
    if (step >= window_start) {
      ++win_steps;
      win_task += task;
      win_aux += aux;
      win_comm += comm;
      for (size_t i = 0; i < dsum.size(); ++i) dsum[i] += counts[i];
      for (int i = 0; i < P; ++i) {
        double row = 0.0, intra = 0.0;
        for (int e = 0; e < N; ++e) row += counts[static_cast<size_t>(i) * N + e];
        for (int dev = 0; dev < P; ++dev) {
          const bool in = o.intra_groups ? o.intra_groups[i * P + dev] != 0 : dev == i;
          if (!in) continue;
          for (int e = dev * E; e < (dev + 1) * E; ++e) intra += counts[static_cast<size_t>(i) * N + e];
        }
        intra_num += intra;
        intra_den += row;
      }
    }
  }
  if (o.steps == 0) {
    rep.initial_dispatch.assign(static_cast<size_t>(P) * N, 0.0);
    rep.final_dispatch.assign(static_cast<size_t>(P) * N, 0.0);
    return rep;
  }
  rep.final_dispatch.resize(dsum.size());
  for (size_t i = 0; i < dsum.size(); ++i) rep.final_dispatch[i] = dsum[i] / static_cast<double>(win_steps);
  rep.final_task_loss = win_task / static_cast<double>(win_steps);
  rep.final_aux_loss = win_aux / static_cast<double>(win_steps);
  rep.final_comm_us = win_comm / static_cast<double>(win_steps);
  rep.intra_share = intra_den > 0.0 ? intra_num / intra_den : 0.0;
  rep.dropped_total_rate = static_cast<double>(dropped_total) / (static_cast<double>(o.steps) * k * S * P);
  const double col_target = static_cast<double>(k) * S * P / N;
  double min_col = std::numeric_limits<double>::infinity();
  for (int e = 0; e < N; ++e) {
    double col = 0.0;
    for (int i = 0; i < P; ++i) col += rep.final_dispatch[static_cast<size_t>(i) * N + e];
    rep.col_balance_max_dev = std::max(rep.col_balance_max_dev, std::abs(col - col_target) / col_target);
    min_col = std::min(min_col, col);
  }
  rep.min_expert_load = min_col;
  if (c_hat) {
    double tv0 = 0.0, tv1 = 0.0;
    for (int i = 0; i < P; ++i) {
      rep.tv_rows.push_back(tv_distance(rep.final_dispatch.data() + static_cast<size_t>(i) * N,
                                        c_hat + static_cast<size_t>(i) * N, N));
      tv0 += tv_distance(rep.initial_dispatch.data() + static_cast<size_t>(i) * N, c_hat + static_cast<size_t>(i) * N,
                         N);
      tv1 += rep.tv_rows.back();
    }
    rep.tv_initial_mean = tv0 / P;
    rep.tv_final_mean = tv1 / P;
  }
  return rep;
}


}  // namespace

TrainReport train_layer(LayerConfig cfg, const double* c_hat, const TrainOptions& o, const __nv_bfloat16* x,
                        const __nv_bfloat16* y, __nv_bfloat16* wg, __nv_bfloat16* w1, __nv_bfloat16* w2,
                        cudaStream_t s) {
  require(cfg.world_size == 1, "train: single-device layer (P logical processes); expert parallelism: "
                               "tamoe_layer_train on a layer created with tamoe_layer_create_ep[_begin]");
  require(o.kind >= 0 && o.kind <= 2, "train: unknown loss kind");
  require(o.kind == 0 || c_hat != nullptr, "topo and compulsory losses require a target pattern");
  cfg.aux_kind = o.kind;  // 2 = compulsory quota routing + balance loss
  require(cfg.N % cfg.P == 0, "N must be divisible by P");
  Layer layer(cfg, cfg.aux_kind != 0 ? c_hat : nullptr);
  return train_on_layer(layer, c_hat, o, x, y, wg, w1, w2, s);
}

TrainReport train_on_layer(Layer& layer, const double* c_hat, const TrainOptions& o, const __nv_bfloat16* x,
                           const __nv_bfloat16* y, __nv_bfloat16* wg, __nv_bfloat16* w1, __nv_bfloat16* w2,
                           cudaStream_t s) {
  const LayerConfig& cfg = layer.cfg();
  require(o.kind >= 0 && o.kind <= 2, "train: unknown loss kind");
  require(o.steps >= 0, "train: steps must be >= 0");
  require(o.kind == 0 || c_hat != nullptr, "topo and compulsory losses require a target pattern");
  require(cfg.aux_kind == o.kind, "train: the layer was created with a different aux loss kind");
  const int W = cfg.world_size, me = cfg.rank;
  const int P = cfg.P, S = cfg.S, N = cfg.N, E = N / W;
  const int Pg = P * W;  // processes of the report (one per rank under expert parallelism)
  require(N % Pg == 0, "N must be divisible by the number of processes");
  const int n_pad = layer.n_pad();
  const long long n_wg = static_cast<long long>(P) * n_pad * cfg.d;
  const long long n_w1 = static_cast<long long>(E) * (cfg.f == 0 ? cfg.d_out : cfg.f) * cfg.d;
  const long long n_w2 = cfg.f == 0 ? 0 : static_cast<long long>(E) * cfg.d_out * cfg.f;

  DevBuf buf;
  float* m_wg = buf.get<float>(n_wg);
  float* m_w1 = buf.get<float>(n_w1);
  float* m_w2 = n_w2 ? buf.get<float>(n_w2) : nullptr;
  widen_bf16(wg, m_wg, n_wg, s);
  widen_bf16(w1, m_w1, n_w1, s);
  if (n_w2) widen_bf16(w2, m_w2, n_w2, s);
  LayerIO io{};
  io.x = x;
  io.y = y;
  io.wg = wg;
  io.w1 = w1;
  io.w2 = n_w2 ? w2 : nullptr;
  io.dwg = buf.get<float>(n_wg);
  io.dw1 = buf.get<__nv_bfloat16>(n_w1);
  io.dw2 = n_w2 ? buf.get<__nv_bfloat16>(n_w2) : nullptr;
  io.dx = cfg.need_dx ? buf.get<__nv_bfloat16>(static_cast<long long>(P) * S * cfg.d) : nullptr;
  io.losses = buf.get<double>(2);

  // per-step CUDA-event phase timing (eager steps): the measured exchange of each step = the counts exchange +
  // dispatch phases under expert parallelism (a2a_counts, a2a_dispatch), the local permute otherwise
  PhaseTimer& tm = layer.timer();
  tm.reset();
  tm.enabled = true;
  std::vector<double> prev(PhaseTimer::kMax, 0.0);
  const RouteBuffers& rb = layer.route().buf;
  const size_t pn = static_cast<size_t>(P) * N;
  const size_t rec = 4 + 2 * pn;  // per rank: task, aux, measured exchange, pad, kept counts, dropped counts
  std::vector<double> mine(rec), all(static_cast<size_t>(W) * rec);
  std::vector<int> cnt_local(pn), drop_local(pn);
  TrainReport rep = run_train(Pg, S, N, cfg.k, cfg.d, cfg.cap_mode, cfg.aux_weight, c_hat, o,
                              [&](int step, double* losses, int* counts_i, int* dropped_i, double* measured) {
    if (o.kind == 1 && o.switch_step != INT_MIN && step > o.switch_step) layer.set_aux_kind(0);
    layer.step(io, s);
    layer.status();  // non-finite logit: ValidationError before the update (gate.cpp:16-17)
    double loc[2];
    TAMOE_CUDA(cudaMemcpyAsync(loc, io.losses, sizeof(double) * 2, cudaMemcpyDeviceToHost, s));
    TAMOE_CUDA(cudaMemcpyAsync(cnt_local.data(), rb.counts, sizeof(int) * pn, cudaMemcpyDeviceToHost, s));
    TAMOE_CUDA(cudaMemcpyAsync(drop_local.data(), rb.dropped, sizeof(int) * pn, cudaMemcpyDeviceToHost, s));
    // synchronized update, fixed order (gates, then experts)
    sgd_step(m_wg, io.dwg, static_cast<float>(o.lr), wg, n_wg, s);
    sgd_step(m_w1, io.dw1, static_cast<float>(o.lr), w1, n_w1, s);
    if (n_w2) sgd_step(m_w2, io.dw2, static_cast<float>(o.lr), w2, n_w2, s);
    TAMOE_CUDA(cudaStreamSynchronize(s));
    tm.fold();
    double comm = 0.0;
    for (int i = 0; i < tm.n; ++i) {
      const std::string nm = tm.names[i];
      const double dt = tm.total_ms[i] - prev[static_cast<size_t>(i)];
      prev[static_cast<size_t>(i)] = tm.total_ms[i];
      if (W > 1 ? (nm == "a2a_counts" || nm == "a2a_dispatch") : nm == "permute") comm += dt * 1e3;
    }
    if (W == 1) {
      losses[0] = loc[0];
      losses[1] = loc[1];
      std::copy(cnt_local.begin(), cnt_local.end(), counts_i);
      std::copy(drop_local.begin(), drop_local.end(), dropped_i);
      *measured = comm;
      return;
    }
    // every rank's losses (its share), kept / dropped counts and measured exchange -> every rank (peer stores +
    // device barrier over the mapped workspaces): the report covers all P processes, identically on every rank
    mine[0] = loc[0];
    mine[1] = loc[1];
    mine[2] = comm;
    mine[3] = 0.0;
    for (size_t i = 0; i < pn; ++i) {
      mine[4 + i] = cnt_local[i];
      mine[4 + pn + i] = drop_local[i];
    }
    layer.allgather_host(mine.data(), static_cast<int>(rec), all.data(), s);
    losses[0] = losses[1] = 0.0;
    *measured = 0.0;
    for (int r = 0; r < W; ++r) {  // rank order: the sums are identical on every rank
      const double* row = all.data() + static_cast<size_t>(r) * rec;
      losses[0] += row[0];
      losses[1] += row[1];
      *measured = std::max(*measured, row[2]);
      for (size_t i = 0; i < pn; ++i) {
        counts_i[static_cast<size_t>(r) * pn + i] = static_cast<int>(row[4 + i]);
        dropped_i[static_cast<size_t>(r) * pn + i] = static_cast<int>(row[4 + pn + i]);
      }
    }
    (void)me;
  });
  tm.enabled = false;
  tm.reset();
  return rep;
}

TrainReport train_f64(int P, int S, int d, int d_out, int N, int k, int cap_mode, double cf, double aux_weight,
                      int norm, double temperature, const double* c_hat, const TrainOptions& o, const double* x,
                      const double* y, double* gates, double* experts, cudaStream_t s) {
  require(o.kind >= 0 && o.kind <= 2, "train: unknown loss kind");
  require(o.steps >= 0, "train: steps must be >= 0");
  require(N % P == 0, "N must be divisible by P");
  require(o.kind == 0 || c_hat != nullptr, "topo and compulsory losses require a target pattern");
  std::vector<double> pen;
  if (c_hat) {
    for (int i = 0; i < P; ++i) {
      const auto row = penalty_weights(c_hat + static_cast<size_t>(i) * N, N, norm, temperature);
      pen.insert(pen.end(), row.begin(), row.end());
    }
  }
  // the reference withholds c_hat from balance routing (trainer.cpp:250)
  const auto caps = capacity_caps(cap_mode, cf, k, S, N, P, o.kind == 0 ? nullptr : c_hat);
  Router router(P, S, N, k);
  DevBuf buf;
  const long long n_g = static_cast<long long>(P) * d * N, n_u = static_cast<long long>(N) * d * d_out;
  double* gg = buf.get<double>(n_g);
  double* eg = buf.get<double>(n_u);
  const RouteBuffers& rb = router.rw.buf;
  return run_train(P, S, N, k, d, cap_mode, aux_weight, c_hat, o,
                   [&](int step, double* losses, int* counts_i, int* dropped_i, double*) {
                     F64StepArgs a;
                     a.d = d;
                     a.d_out = d_out;
                     a.x = x;
                     a.y = y;
                     a.gates = gates;
                     a.experts = experts;
                     const bool switched = o.kind == 1 && o.switch_step != INT_MIN && step > o.switch_step;
                     a.aux_kind = switched ? 0 : o.kind;
                     a.penalty = pen.empty() ? nullptr : pen.data();
                     a.c_hat = c_hat;
                     a.aux_weight = aux_weight;
                     a.cap_mode = cap_mode;
                     a.caps = caps.data();
                     a.gate_grads = gg;
                     a.expert_grads = eg;
                     a.losses = losses;
                     layer_step_f64(router.rw, a, s);
                     const size_t pn = static_cast<size_t>(P) * N;
                     TAMOE_CUDA(cudaMemcpyAsync(counts_i, rb.counts, sizeof(int) * pn, cudaMemcpyDeviceToHost, s));
                     TAMOE_CUDA(cudaMemcpyAsync(dropped_i, rb.dropped, sizeof(int) * pn, cudaMemcpyDeviceToHost, s));
                     // synchronized update, fixed order (gates, then experts), in the reference's rounding
                     sgd_step_f64(gates, gg, o.lr, n_g, s);
                     sgd_step_f64(experts, eg, o.lr, n_u, s);
                     TAMOE_CUDA(cudaStreamSynchronize(s));
                   });
}

}  // namespace tamoe
