// extern "C" boundary (include/tamoe.h).  Each entry point translates C++
// exceptions into the reference's status convention via guarded().
#include "../../include/tamoe.h"

#include <algorithm>
#include <climits>
#include <memory>
#include <string>
#include <vector>
#include <cstring>

#include "capi_util.hpp"
#include "ep.hpp"
#include "expert.hpp"
#include "gate.hpp"
#include "gate_f64.hpp"
#include "layer_f64.hpp"
#include "host_topology.hpp"
#include "layer.hpp"
#include "route.hpp"
#include "trainer.hpp"

using namespace tamoe;

struct tamoe_router {
  Router impl;
  tamoe_router(int P, int S, int N, int k) : impl(P, S, N, k) {}
};
struct tamoe_layer {
  Layer impl;
  tamoe_layer(const LayerConfig& c, const double* ch, std::unique_ptr<EpComm> ep = nullptr)
      : impl(c, ch, std::move(ep)) {}
};
struct tamoe_p2p_probe {
  P2PProbe impl;
  tamoe_p2p_probe(std::unique_ptr<EpComm> c, size_t bytes) : impl(std::move(c), bytes) {}
};

namespace {

struct ReadSpec {
  const void* src;
  long long bytes;
};

ReadSpec route_array(const RouteWorkspace& rw, int what, const float* logits) {
  const RouteDims& d = rw.dims;
  const RouteBuffers& b = rw.buf;
  const long long picks = d.picks(), pn = static_cast<long long>(d.P) * d.N;
  switch (what) {
    case TAMOE_R_IDX: return {b.idx, picks * 4};
    case TAMOE_R_GATE: return {b.gate, picks * 4};
    case TAMOE_R_SCORE: return {b.score, picks * 8};
    case TAMOE_R_KEPT: return {b.kept, picks};
    case TAMOE_R_POS: return {b.pos, picks * 4};
    case TAMOE_R_COUNTS: return {b.counts, pn * 4};
    case TAMOE_R_DROPPED: return {b.dropped, pn * 4};
    case TAMOE_R_MEAN_PROBS: return {b.mean_probs, pn * 8};
    case TAMOE_R_SEG_START: return {b.seg_start, d.N * 4LL};
    case TAMOE_R_SEG_ROWS: return {b.seg_rows, d.N * 4LL};
    case TAMOE_R_CLIST: return {b.clist, picks * 4};
    case TAMOE_R_LIST_START: return {b.list_start, d.N * 4LL};
    case TAMOE_R_BAD: return {b.bad, 4};
    case TAMOE_R_GATE64:
      require(b.gate64 != nullptr, "fp64 gate values are only kept by the standalone router");
      return {b.gate64, picks * 8};
    case TAMOE_R_LOGITS:
      require(logits != nullptr, "logits are only kept by the layer");
      return {logits, static_cast<long long>(d.P) * d.S * d.N * 4};
    default: throw ValidationError("unknown routing array id");
  }
}

void read_array(const RouteWorkspace& rw, int what, void* dst, long long bytes, cudaStream_t s, const float* lg) {
  ReadSpec r = route_array(rw, what, lg);
  require(dst != nullptr && bytes >= r.bytes, "read: destination too small");
  TAMOE_CUDA(cudaMemcpyAsync(dst, r.src, r.bytes, cudaMemcpyDefault, s));
  TAMOE_CUDA(cudaStreamSynchronize(s));
}

// Stream-ordered device scratch for the fp64 operators.
template <class T>
struct DeviceScratch {
  T* p = nullptr;
  cudaStream_t s;
  DeviceScratch(long long n, cudaStream_t st) : s(st) {
    TAMOE_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * (n > 0 ? n : 1), s));
  }
  ~DeviceScratch() { cudaFreeAsync(p, s); }
  T read(cudaStream_t st) const {
    T v{};
    TAMOE_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, st));
    TAMOE_CUDA(cudaStreamSynchronize(st));
    return v;
  }
};

void check_bad(const RouteWorkspace& rw, cudaStream_t s) {
  int bad = 0;
  TAMOE_CUDA(cudaMemcpyAsync(&bad, rw.buf.bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  TAMOE_CUDA(cudaStreamSynchronize(s));
  require(bad == 0, "non-finite gate logit");
}

}  // namespace

extern "C" {

const char* tamoe_last_error(void) { return last_error_slot().c_str(); }
int tamoe_version(void) { return 1; }

int tamoe_largest_remainder_round(const double* values, int n, long long target, long long* out) {
  return guarded([&] {
    require(n >= 0 && (n == 0 || (values && out)), "largest_remainder_round: null buffer");
    auto r = largest_remainder_round(values, n, target);
    if (n) std::memcpy(out, r.data(), sizeof(long long) * n);
  });
}

int tamoe_penalty_weights(const double* c_hat_row, int n, int norm, double temperature, double* p) {
  return guarded([&] {
    require(n >= 1 && c_hat_row && p, "penalty_weights: empty row");
    require(norm == TAMOE_NORM_SUM || norm == TAMOE_NORM_SOFTMAX, "unknown penalty normalization");
    auto r = penalty_weights(c_hat_row, n, norm, temperature);
    std::memcpy(p, r.data(), sizeof(double) * n);
  });
}

int tamoe_target_closed_form(const double* beta_hat, int P, int N, int k, int S, double* c_hat) {
  return guarded([&] {
    require(beta_hat && c_hat, "target_closed_form: null buffer");
    auto r = target_closed_form(beta_hat, P, N, k, S);
    std::memcpy(c_hat, r.data(), sizeof(double) * r.size());
  });
}

int tamoe_capacity_caps(int mode, double capacity_factor, int k, int S, int N, int P, const double* c_hat,
                        long long* caps) {
  return guarded([&] {
    require(caps && P >= 1 && N >= 1 && S >= 0, "capacity_caps: bad shape");
    auto r = capacity_caps(mode, capacity_factor, k, S, N, P, c_hat);
    std::memcpy(caps, r.data(), sizeof(long long) * r.size());
  });
}

int tamoe_device_payload_tokens(const double* counts, int P, int N, double* payload) {
  return guarded([&] {
    require(counts && payload, "device_payload_tokens: null buffer");
    auto r = device_payload_tokens(counts, P, N);
    std::memcpy(payload, r.data(), sizeof(double) * r.size());
  });
}

int tamoe_fit_profile(const int* src, const int* dst, const double* message_mb, const double* time_us, int n,
                      int P, double* alpha, double* beta) {
  return guarded([&] {
    require(src && dst && message_mb && time_us && alpha && beta, "fit_profile: null buffer");
    fit_profile(src, dst, message_mb, time_us, n, P, alpha, beta);
  });
}

int tamoe_fill_partial_profile(const double* alpha, const double* beta, int P, const int* levels, int n_levels,
                               double self_beta_floor, double* alpha_out, double* beta_out) {
  return guarded([&] {
    require(alpha && beta && alpha_out && beta_out, "fill_partial_profile: null buffer");
    fill_partial_profile(alpha, beta, P, levels, n_levels, self_beta_floor, alpha_out, beta_out);
  });
}

int tamoe_smooth_profile(const int* levels, int n_levels, const double* alpha, const double* beta, int P,
                         double self_beta_floor, double* alpha_hat, double* beta_hat, double* level_alpha,
                         double* level_beta) {
  return guarded([&] {
    require(alpha && beta && alpha_hat && beta_hat, "smooth_profile: null buffer");
    std::vector<double> la, lb;
    smooth_profile(levels, n_levels, alpha, beta, P, self_beta_floor, alpha_hat, beta_hat, &la, &lb);
    if (level_alpha) std::copy(la.begin(), la.end(), level_alpha);
    if (level_beta) std::copy(lb.begin(), lb.end(), level_beta);
  });
}

int tamoe_exchange_cost(const double* alpha, const double* beta, const double* c, int P, int N, int d, int b,
                        int extra_alpha_rounds, double* pair_cost_us, double* summary) {
  return guarded([&] {
    require(alpha && beta && c && summary, "exchange_cost: null buffer");
    const ExchangeCost r = exchange_cost(alpha, beta, c, P, N, d, b, extra_alpha_rounds);
    if (pair_cost_us) std::copy(r.pair_cost_us.begin(), r.pair_cost_us.end(), pair_cost_us);
    summary[0] = r.bottleneck_us;
    summary[1] = r.total_bytes;
    summary[2] = r.size_exchange_us;
    summary[3] = r.total_estimate_us;
  });
}

int tamoe_grouped_fwd(const void* tokens, const void* w, int G, int M, int K, int R, const int* seg_start,
                      const int* seg_rows, void* out, void* pre_out, int act, void* stream) {
  return guarded([&] {
    grouped_fwd(static_cast<const __nv_bfloat16*>(tokens), static_cast<const __nv_bfloat16*>(w), G, M, K, R,
                seg_start, seg_rows, static_cast<__nv_bfloat16*>(out), static_cast<__nv_bfloat16*>(pre_out), act,
                static_cast<cudaStream_t>(stream));
  });
}

int tamoe_grouped_dgrad(const void* grad_tokens, const void* w, int G, int M, int K, int R, const int* seg_start,
                        const int* seg_rows, void* out, const void* pre_in, int act, void* stream) {
  return guarded([&] {
    grouped_dgrad(static_cast<const __nv_bfloat16*>(grad_tokens), static_cast<const __nv_bfloat16*>(w), G, M, K, R,
                  seg_start, seg_rows, static_cast<__nv_bfloat16*>(out),
                  static_cast<const __nv_bfloat16*>(pre_in), act, static_cast<cudaStream_t>(stream));
  });
}

int tamoe_grouped_wgrad(const void* a_tokens, const void* b_tokens, int G, int M, int N, int R,
                        const int* seg_start, const int* seg_rows, void* out, void* stream) {
  return guarded([&] {
    grouped_wgrad(static_cast<const __nv_bfloat16*>(a_tokens), static_cast<const __nv_bfloat16*>(b_tokens), G, M, N,
                  R, seg_start, seg_rows, static_cast<__nv_bfloat16*>(out), static_cast<cudaStream_t>(stream));
  });
}

int tamoe_router_create(int P, int S, int N, int k, tamoe_router** out) {
  return guarded([&] {
    require(out != nullptr, "router_create: null out");
    *out = new tamoe_router(P, S, N, k);
  });
}

int tamoe_router_destroy(tamoe_router* r) {
  return guarded([&] { delete r; });
}

int tamoe_router_route_probs(tamoe_router* r, const double* probs, int mode, const long long* caps, void* stream) {
  return guarded([&] {
    require(r && probs && caps, "route_probs: null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    RouteWorkspace& rw = r->impl.rw;
    rw.upload_caps(caps, s);
    route_rows_from_probs(probs, rw.dims, rw.row_out(nullptr, nullptr), s);
    rw.finish(mode, s);
  });
}

int tamoe_router_route_gate(tamoe_router* r, const void* x, const void* wg, int n_pad, int d, float* logits,
                            double* probs, int mode, const long long* caps, void* stream) {
  return guarded([&] {
    require(r && x && wg && caps, "route_gate: null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    RouteWorkspace& rw = r->impl.rw;
    rw.upload_caps(caps, s);
    TAMOE_CUDA(cudaMemsetAsync(rw.buf.bad, 0, sizeof(int), s));
    gate_forward(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(wg), n_pad, rw.dims, d,
                 rw.row_out(logits ? logits : rw.buf.logits, probs), s);
    check_bad(rw, s);
    rw.finish(mode, s);
  });
}

int tamoe_router_permute(tamoe_router* r, const void* x, int d, void* xp, int r_max, void* stream) {
  return guarded([&] {
    require(r && x && xp, "permute: null argument");
    RouteWorkspace& rw = r->impl.rw;
    PeerBufs pb{};
    pb.p[0] = static_cast<__nv_bfloat16*>(xp);
    route_permute(rw.dims, rw.buf, static_cast<const __nv_bfloat16*>(x), d, pb, r_max, nullptr, 0, RowMap{},
                  static_cast<cudaStream_t>(stream));
  });
}

int tamoe_router_read(tamoe_router* r, int what, void* dst, long long bytes, void* stream) {
  return guarded([&] {
    require(r != nullptr, "read: null router");
    read_array(r->impl.rw, what, dst, bytes, static_cast<cudaStream_t>(stream), nullptr);
  });
}

int tamoe_softmax_rows_f64(const double* logits, int rows, int cols, double* probs, void* stream) {
  return guarded([&] {
    require(rows >= 0 && cols >= 0 && (rows * static_cast<long long>(cols) == 0 || (logits && probs)),
            "softmax_rows: null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DeviceScratch<int> bad(1, s);
    TAMOE_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    softmax_rows_f64(logits, probs, rows, cols, bad.p, s);
    require(bad.read(s) == 0, "non-finite gate logit");
  });
}

int tamoe_gate_forward_f64(const double* x, const double* w, int S, int d, int N, double* probs, void* stream) {
  return guarded([&] {
    require(S >= 0 && d >= 0 && N >= 0, "gate_forward: negative shape");
    if (static_cast<long long>(S) * N == 0) return;
    require(x && w && probs, "gate_forward: null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    matmul_f64(x, w, probs, S, N, d, s);  // logits in place, then the row softmax
    DeviceScratch<int> bad(1, s);
    TAMOE_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    softmax_rows_f64(probs, probs, S, N, bad.p, s);
    require(bad.read(s) == 0, "non-finite gate logit");
  });
}

int tamoe_grad_aux_loss_f64(const double* x, const double* probs, const double* coeff, int S, int d, int N,
                            double* grad, void* stream) {
  return guarded([&] {
    require(S >= 0 && d >= 0 && N >= 0, "grad_aux_loss: negative shape");
    if (static_cast<long long>(d) * N == 0) return;
    require(grad && coeff && (S == 0 || (x && probs)), "grad_aux_loss: null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    TAMOE_CUDA(cudaMemsetAsync(grad, 0, sizeof(double) * d * N, s));
    if (S == 0) return;
    DeviceScratch<double> c(N, s), dz(static_cast<long long>(S) * N, s);
    TAMOE_CUDA(cudaMemcpyAsync(c.p, coeff, sizeof(double) * N, cudaMemcpyHostToDevice, s));
    aux_dz_f64(probs, c.p, dz.p, S, N, s);
    add_atb_f64(grad, x, dz.p, S, d, N, s);
    TAMOE_CUDA(cudaStreamSynchronize(s));  // coeff is the caller's host memory
  });
}

int tamoe_layer_step_f64(tamoe_router* r, int d, int d_out, const double* x, const double* y, const double* gates,
                         const double* experts, const double* penalty, const double* c_hat, int aux_kind,
                         double aux_weight, int cap_mode, const long long* caps, double* probs, double* gate_grads,
                         double* expert_grads, double* y_hat, double* losses, void* stream) {
  return guarded([&] {
    require(r != nullptr, "layer_step_f64: null router");
    F64StepArgs a;
    a.d = d;
    a.d_out = d_out;
    a.x = x;
    a.y = y;
    a.gates = gates;
    a.experts = experts;
    a.penalty = penalty;
    a.c_hat = c_hat;
    a.aux_kind = aux_kind;
    a.aux_weight = aux_weight;
    a.cap_mode = cap_mode;
    a.caps = caps;
    a.probs = probs;
    a.gate_grads = gate_grads;
    a.expert_grads = expert_grads;
    a.y_hat = y_hat;
    a.losses = losses;
    layer_step_f64(r->impl.rw, a, static_cast<cudaStream_t>(stream));
  });
}

int tamoe_loss_balance(const long long* counts, const double* mean_probs, int N, int S, double* loss) {
  return guarded([&] {
    require(N >= 0 && (N == 0 || (counts && mean_probs)) && loss, "loss_balance: null buffer");
    *loss = loss_balance(counts, mean_probs, N, S);
  });
}

int tamoe_loss_topo(const long long* counts, const double* mean_probs, const double* penalty, int n, int N, int P,
                    int S, double* loss) {
  return guarded([&] {
    require(n >= 0 && (n == 0 || (counts && mean_probs && penalty)) && loss, "loss_topo: null buffer");
    *loss = loss_topo(counts, mean_probs, penalty, n, N, P, S);
  });
}

int tamoe_aux_coefficients(int kind, const long long* counts, const double* penalty, int n, int N, int P, int S,
                           double* coeff) {
  return guarded([&] {
    require(n >= 0 && (n == 0 || (counts && coeff)), "aux_coefficients: null buffer");
    require(kind == TAMOE_LOSS_BALANCE || kind == TAMOE_LOSS_TOPO, "unknown aux loss kind");
    auto c = aux_coefficients(kind, counts, penalty, n, N, P, S);
    if (n) std::memcpy(coeff, c.data(), sizeof(double) * n);
  });
}

int tamoe_layer_create(const tamoe_layer_config* cfg, const double* c_hat, tamoe_layer** out) {
  return guarded([&] {
    require(cfg && out, "layer_create: null argument");
    LayerConfig c{cfg->P, cfg->S, cfg->d, cfg->d_out, cfg->N, cfg->k, cfg->f, cfg->act, cfg->cap_mode,
                  cfg->capacity_factor, cfg->aux_kind, cfg->aux_weight, cfg->penalty_norm, cfg->temperature,
                  cfg->need_dx, cfg->world_size, cfg->rank};
    *out = new tamoe_layer(c, c_hat);
  });
}

namespace {

TrainOptions train_options(const tamoe_train_opts* opts) {
  TrainOptions o;
  o.kind = opts->kind;
  o.steps = opts->steps;
  o.lr = opts->lr;
  o.switch_step = opts->has_switch ? opts->switch_step : INT_MIN;
  o.report_window = opts->report_window;
  o.bytes_per_element = opts->bytes_per_element;
  o.alpha_hat = opts->alpha_hat;
  o.beta_hat = opts->beta_hat;
  o.intra_groups = opts->intra_groups;
  return o;
}

void fill_report(const TrainReport& r, tamoe_train_report* report) {
  auto put = [](double* dst, const std::vector<double>& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(double) * v.size());
  };
  put(report->task_loss, r.task_loss);
  put(report->aux_loss, r.aux_loss);
  put(report->comm_us, r.comm_us);
  put(report->dropped_rate, r.dropped_rate);
  put(report->initial_dispatch, r.initial_dispatch);
  put(report->final_dispatch, r.final_dispatch);
  put(report->tv_rows, r.tv_rows);
  put(report->comm_measured_us, r.comm_measured_us);
  const double sm[9] = {r.tv_initial_mean, r.tv_final_mean, r.col_balance_max_dev, r.min_expert_load,
                        r.intra_share, r.final_task_loss, r.final_aux_loss, r.final_comm_us, r.dropped_total_rate};
  std::memcpy(report->summary, sm, sizeof(sm));
}

}  // namespace

int tamoe_train(const tamoe_layer_config* cfg, const double* c_hat, const tamoe_train_opts* opts, const void* x,
                const void* y, void* wg, void* w1, void* w2, tamoe_train_report* report, void* stream) {
  return guarded([&] {
    require(cfg && opts && x && y && wg && w1 && report, "train: null argument");
    require(cfg->f == 0 || w2, "train: FFN experts need w2");
    LayerConfig c{cfg->P, cfg->S, cfg->d, cfg->d_out, cfg->N, cfg->k, cfg->f, cfg->act, cfg->cap_mode,
                  cfg->capacity_factor, cfg->aux_kind, cfg->aux_weight, cfg->penalty_norm, cfg->temperature,
                  cfg->need_dx, cfg->world_size, cfg->rank};
    const TrainReport r = train_layer(c, c_hat, train_options(opts), static_cast<const __nv_bfloat16*>(x),
                                      static_cast<const __nv_bfloat16*>(y), static_cast<__nv_bfloat16*>(wg),
                                      static_cast<__nv_bfloat16*>(w1), static_cast<__nv_bfloat16*>(w2),
                                      static_cast<cudaStream_t>(stream));
    fill_report(r, report);
  });
}

int tamoe_layer_train(tamoe_layer* l, const double* c_hat, const tamoe_train_opts* opts, const void* x, const void* y,
                      void* wg, void* w1, void* w2, tamoe_train_report* report, void* stream) {
  return guarded([&] {
    require(l && opts && x && y && wg && w1 && report, "layer_train: null argument");
    require(l->impl.cfg().f == 0 || w2, "layer_train: FFN experts need w2");
    const TrainReport r = train_on_layer(l->impl, c_hat, train_options(opts), static_cast<const __nv_bfloat16*>(x),
                                         static_cast<const __nv_bfloat16*>(y), static_cast<__nv_bfloat16*>(wg),
                                         static_cast<__nv_bfloat16*>(w1), static_cast<__nv_bfloat16*>(w2),
                                         static_cast<cudaStream_t>(stream));
    fill_report(r, report);
  });
}

int tamoe_train_f64(const tamoe_layer_config* cfg, const double* c_hat, const tamoe_train_opts* opts,
                    const double* x, const double* y, double* gates, double* experts, tamoe_train_report* report,
                    void* stream) {
  return guarded([&] {
    require(cfg && opts && report && gates && experts, "train_f64: null argument");
    require(cfg->P >= 1 && cfg->S >= 0 && cfg->d >= 1 && cfg->d_out >= 1 && cfg->N >= 1, "train_f64: bad shape");
    require(static_cast<long long>(cfg->P) * cfg->S == 0 || (x && y), "train_f64: null batch");
    const TrainReport r = train_f64(cfg->P, cfg->S, cfg->d, cfg->d_out, cfg->N, cfg->k, cfg->cap_mode,
                                    cfg->capacity_factor, cfg->aux_weight, cfg->penalty_norm, cfg->temperature, c_hat,
                                    train_options(opts), x, y, gates, experts, static_cast<cudaStream_t>(stream));
    fill_report(r, report);
  });
}

int tamoe_p2p_sweep(const void* nccl_id128, int world, int rank, const double* sizes_mb, int nsizes, int reps,
                    int warmup, double* time_us) {
  return guarded([&] {
    require(nccl_id128 && sizes_mb && time_us, "p2p_sweep: null argument");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id128, sizeof(id));
    double max_mb = 0.0;
    for (int i = 0; i < nsizes; ++i) max_mb = std::max(max_mb, sizes_mb[i]);
    P2PProbe probe(std::make_unique<EpComm>(world, rank, id),
                   (static_cast<size_t>(max_mb * 1e6) + 4095) & ~static_cast<size_t>(4095));
    const std::vector<double> t = probe.sweep(sizes_mb, nsizes, reps, warmup);
    std::memcpy(time_us, t.data(), sizeof(double) * t.size());
  });
}

int tamoe_set_link_emulation(int group_size, int repeat) {
  return guarded([&] {
    require(group_size >= 0 && repeat >= 1 && repeat <= 255, "link emulation: group_size >= 0, repeat in [1, 255]");
    link_emulation().group_size = group_size;
    link_emulation().repeat = repeat;
  });
}

int tamoe_nccl_unique_id(void* out128) {
  return guarded([&] {
    require(out128 != nullptr, "nccl_unique_id: null output");
    static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw std::runtime_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out128, &id, sizeof(id));
  });
}

int tamoe_layer_create_ep(const tamoe_layer_config* cfg, const double* c_hat, const void* nccl_id128,
                          tamoe_layer** out) {
  return guarded([&] {
    require(cfg && out && nccl_id128, "layer_create_ep: null argument");
    LayerConfig c{cfg->P, cfg->S, cfg->d, cfg->d_out, cfg->N, cfg->k, cfg->f, cfg->act, cfg->cap_mode,
                  cfg->capacity_factor, cfg->aux_kind, cfg->aux_weight, cfg->penalty_norm, cfg->temperature,
                  cfg->need_dx, cfg->world_size, cfg->rank};
    ncclUniqueId id;
    std::memcpy(&id, nccl_id128, sizeof(id));
    auto ep = std::make_unique<EpComm>(c.world_size, c.rank, id);
    *out = new tamoe_layer(c, c_hat, std::move(ep));
  });
}

int tamoe_layer_create_ep_begin(const tamoe_layer_config* cfg, const double* c_hat, tamoe_layer** out,
                                void* blob_out) {
  return guarded([&] {
    require(cfg && out && blob_out, "layer_create_ep_begin: null argument");
    LayerConfig c{cfg->P, cfg->S, cfg->d, cfg->d_out, cfg->N, cfg->k, cfg->f, cfg->act, cfg->cap_mode,
                  cfg->capacity_factor, cfg->aux_kind, cfg->aux_weight, cfg->penalty_norm, cfg->temperature,
                  cfg->need_dx, cfg->world_size, cfg->rank};
    auto l = std::make_unique<tamoe_layer>(c, c_hat, std::make_unique<EpComm>(c.world_size, c.rank));
    const PeerBlob b = l->impl.blob();
    std::memcpy(blob_out, &b, sizeof(b));
    *out = l.release();
  });
}

int tamoe_layer_ep_connect(tamoe_layer* l, const void* blobs) {
  return guarded([&] {
    require(l && blobs, "layer_ep_connect: null argument");
    const int W = l->impl.cfg().world_size;
    std::vector<PeerBlob> all(static_cast<size_t>(W));
    std::memcpy(all.data(), blobs, sizeof(PeerBlob) * all.size());
    l->impl.connect(all.data());
  });
}

int tamoe_p2p_probe_create(int world, int rank, double max_mb, tamoe_p2p_probe** out, void* blob_out) {
  return guarded([&] {
    require(out && blob_out && max_mb > 0.0, "p2p_probe_create: bad argument");
    auto p = std::make_unique<tamoe_p2p_probe>(std::make_unique<EpComm>(world, rank),
                                               (static_cast<size_t>(max_mb * 1e6) + 4095) & ~static_cast<size_t>(4095));
    const PeerBlob b = p->impl.blob();
    std::memcpy(blob_out, &b, sizeof(b));
    *out = p.release();
  });
}

int tamoe_p2p_probe_connect(tamoe_p2p_probe* p, const void* blobs, int world) {
  return guarded([&] {
    require(p && blobs && world >= 1 && world <= kMaxRanks, "p2p_probe_connect: bad argument");
    std::vector<PeerBlob> all(static_cast<size_t>(world));
    std::memcpy(all.data(), blobs, sizeof(PeerBlob) * all.size());
    p->impl.connect(all.data());
  });
}

int tamoe_p2p_probe_sweep(tamoe_p2p_probe* p, const double* sizes_mb, int nsizes, int reps, int warmup,
                          double* time_us) {
  return guarded([&] {
    require(p && sizes_mb && time_us, "p2p_probe_sweep: null argument");
    const std::vector<double> t = p->impl.sweep(sizes_mb, nsizes, reps, warmup);
    std::memcpy(time_us, t.data(), sizeof(double) * t.size());
  });
}

int tamoe_p2p_probe_destroy(tamoe_p2p_probe* p) {
  return guarded([&] { delete p; });
}

int tamoe_layer_a2a_bytes(tamoe_layer* l, long long* out4) {
  return guarded([&] {
    require(l && out4, "a2a_bytes: null argument");
    l->impl.a2a_bytes(out4);
  });
}

int tamoe_ep_plan(int P, int E, const long long* recv, int* seg_start, int* seg_rows, long long* src_off) {
  return guarded([&] {
    require(P >= 1 && E >= 1 && recv && seg_start && seg_rows && src_off, "ep_plan: bad arguments");
    ep_plan(P, E, recv, seg_start, seg_rows, src_off);
  });
}

int tamoe_layer_destroy(tamoe_layer* l) {
  return guarded([&] { delete l; });
}

int tamoe_layer_step(tamoe_layer* l, const tamoe_layer_io* io, void* stream) {
  return guarded([&] {
    require(l && io, "layer_step: null argument");
    LayerIO x{static_cast<const __nv_bfloat16*>(io->x), static_cast<const __nv_bfloat16*>(io->y),
              static_cast<const __nv_bfloat16*>(io->wg), static_cast<const __nv_bfloat16*>(io->w1),
              static_cast<const __nv_bfloat16*>(io->w2), io->dwg, static_cast<__nv_bfloat16*>(io->dw1),
              static_cast<__nv_bfloat16*>(io->dw2), static_cast<__nv_bfloat16*>(io->dx),
              static_cast<__nv_bfloat16*>(io->y_hat), io->losses};
    l->impl.step(x, static_cast<cudaStream_t>(stream));
  });
}

int tamoe_layer_status(tamoe_layer* l) {
  return guarded([&] {
    require(l != nullptr, "status: null layer");
    l->impl.status();
  });
}

int tamoe_layer_read(tamoe_layer* l, int what, void* dst, long long bytes, void* stream) {
  return guarded([&] {
    require(l != nullptr, "read: null layer");
    read_array(l->impl.route(), what, dst, bytes, static_cast<cudaStream_t>(stream), l->impl.logits());
  });
}

int tamoe_layer_n_pad(int N) { return (N + 15) & ~15; }

int tamoe_layer_launches_per_step(tamoe_layer* l) { return l ? l->impl.launches_per_step() : -1; }

int tamoe_layer_enable_timing(tamoe_layer* l, int enable) {
  return guarded([&] {
    require(l != nullptr, "null layer");
    PhaseTimer& t = l->impl.timer();
    t.reset();
    t.enabled = enable != 0;
  });
}

int tamoe_layer_timing(tamoe_layer* l, const char** names, double* ms, int cap, int* n, int* steps) {
  return guarded([&] {
    require(l && names && ms && n && steps, "timing: null argument");
    PhaseTimer& t = l->impl.timer();
    t.fold();
    const int m = std::min(cap, t.n);
    for (int i = 0; i < m; ++i) {
      names[i] = t.names[i];
      ms[i] = t.total_ms[i];
    }
    *n = m;
    *steps = t.steps;
  });
}

}  // extern "C"
