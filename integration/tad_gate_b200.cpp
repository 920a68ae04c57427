// Drop-in replacement for the reference's proj/core/src/gate.cpp, backed by the B200 library.
//
// A maintainer swaps this file for gate.cpp in the reference's `tadispatch` library (same header,
// tadispatch/gate.hpp:22-97, same value semantics, same exceptions) and links libtamoe.so + cudart; every
// existing caller -- train() (trainer.cpp:243-355), the CLI and the reference's own unit tests -- then runs
// its gate on the GPU:
//
//   gate.hpp symbol                     -> C ABI (include/tamoe.h)               where it runs
//   softmax_rows (gate.cpp:12-28)       -> tamoe_softmax_rows_f64                device, fp64
//   gate_forward (gate.cpp:30-32)       -> tamoe_gate_forward_f64                device, fp64 (bit-identical matmul)
//   topk_route (gate.cpp:91-207)        -> tamoe_capacity_caps + tamoe_router_*  device (top-k, buckets, capacity)
//   largest_remainder_round (:52-78)    -> tamoe_largest_remainder_round         host (once per topology)
//   loss_balance / loss_topo            -> tamoe_loss_balance / tamoe_loss_topo  host (N-vectors)
//   penalty_weights (:222-246)          -> tamoe_penalty_weights                 host (once per topology)
//   *_coefficients, grad_* (:257-296)   -> tamoe_aux_coefficients + tamoe_grad_aux_loss_f64   device, fp64
//   capacity_mode_from_string / to_string / penalty_norm_from_string: string parsing, kept in C++ here.
//
// Status 2 from the library is rethrown as tad::ValidationError, anything else as std::runtime_error --
// the reference's error classes (errors.hpp:11-14).  Built by oracle/ref.mk (`make -f oracle/ref.mk
// suite_b200`) together with the reference's own unit suite; compiled against the reference's headers,
// which are not part of this repository.
#include <cuda_runtime.h>

#include <array>
#include <cmath>
#include <map>
#include <memory>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "tadispatch/errors.hpp"
#include "tadispatch/gate.hpp"
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

// Grow-only device scratch slots, one set per host thread: the reference calls the gate operators many
// times per train() step, so buffers (and routers, below) are reused instead of cudaMalloc/cudaFree per call.
enum Slot { kX, kW, kP, kG, kSlots };
struct Scratch {
  void* p[kSlots] = {};
  size_t cap[kSlots] = {};
  ~Scratch() {
    for (void* q : p) cudaFree(q);
  }
  template <class T>
  T* get(Slot s, size_t n) {
    const size_t bytes = sizeof(T) * (n ? n : 1);
    if (bytes > cap[s]) {
      cudaFree(p[s]);
      p[s] = nullptr;
      cuda(cudaMalloc(&p[s], bytes));
      cap[s] = bytes;
    }
    return static_cast<T*>(p[s]);
  }
};
Scratch& scratch() {
  static thread_local Scratch s;
  return s;
}

template <class T>
T* upload(Slot s, const T* host, size_t n) {
  T* d = scratch().get<T>(s, n);
  if (n) cuda(cudaMemcpy(d, host, sizeof(T) * n, cudaMemcpyHostToDevice));
  return d;
}

template <class T>
void download(T* host, const T* dev, size_t n) {
  if (n) cuda(cudaMemcpy(host, dev, sizeof(T) * n, cudaMemcpyDeviceToHost));
}

struct Router {
  tamoe_router* r = nullptr;
  Router(int P, int S, int N, int k) { check(tamoe_router_create(P, S, N, k, &r)); }
  ~Router() { tamoe_router_destroy(r); }
  Router(const Router&) = delete;
  Router& operator=(const Router&) = delete;
  template <class T>
  std::vector<T> read(int what, size_t n) {
    std::vector<T> v(n);
    check(tamoe_router_read(r, what, v.data(), static_cast<long long>(sizeof(T) * (n ? n : 1)), nullptr));
    return v;
  }
};

// Routers keyed by shape (workspaces are sized at creation), per host thread.
Router& router_for(int P, int S, int N, int k) {
  static thread_local std::map<std::array<int, 4>, std::unique_ptr<Router>> cache;
  auto& slot = cache[{P, S, N, k}];
  if (!slot) {
    if (cache.size() > 64) {  // bound the cache: shapes change rarely in practice
      cache.clear();
      return router_for(P, S, N, k);
    }
    slot = std::make_unique<Router>(P, S, N, k);
  }
  return *slot;
}

int cap_mode(CapacityMode m) {
  switch (m) {
    case CapacityMode::none: return TAMOE_CAP_NONE;
    case CapacityMode::global: return TAMOE_CAP_GLOBAL;
    case CapacityMode::local: return TAMOE_CAP_LOCAL;
    case CapacityMode::local_proportional: return TAMOE_CAP_PROPORTIONAL;
  }
  throw ValidationError("unknown capacity mode");
}

}  // namespace

Matrix softmax_rows(const Matrix& logits) {
  Matrix probs(logits.rows(), logits.cols());
  const size_t n = logits.data().size();
  if (n == 0) return probs;
  double* d = upload(kP, logits.data().data(), n);
  check(tamoe_softmax_rows_f64(d, logits.rows(), logits.cols(), d, nullptr));
  download(probs.data().data(), d, n);
  return probs;
}

Matrix gate_forward(const Matrix& x, const Matrix& W) {
  if (x.cols() != W.rows()) throw ValidationError("gate_forward: x columns must match W rows");
  Matrix probs(x.rows(), W.cols());
  if (probs.data().empty()) return probs;
  const double* dx = upload(kX, x.data().data(), x.data().size());
  const double* dw = upload(kW, W.data().data(), W.data().size());
  double* dp = scratch().get<double>(kP, probs.data().size());
  check(tamoe_gate_forward_f64(dx, dw, x.rows(), x.cols(), W.cols(), dp, nullptr));
  download(probs.data().data(), dp, probs.data().size());
  return probs;
}

CapacityMode capacity_mode_from_string(const std::string& s) {
  if (s == "none") return CapacityMode::none;
  if (s == "global") return CapacityMode::global;
  if (s == "local") return CapacityMode::local;
  if (s == "proportional" || s == "local_proportional") return CapacityMode::local_proportional;
  throw ValidationError("unknown capacity mode: " + s);
}

std::string to_string(CapacityMode mode) {
  switch (mode) {
    case CapacityMode::none: return "none";
    case CapacityMode::global: return "global";
    case CapacityMode::local: return "local";
    case CapacityMode::local_proportional: return "proportional";
  }
  return "unknown";
}

std::vector<RoutingResult> topk_route(const std::vector<Matrix>& probs_per_process, int k,
                                      const CapacityPolicy& policy, const Matrix* c_hat) {
  // validation in the reference's order (gate.cpp:93-107)
  if (probs_per_process.empty()) throw ValidationError("topk_route needs at least one process");
  const int P = static_cast<int>(probs_per_process.size());
  const int N = probs_per_process[0].cols();
  const int S = probs_per_process[0].rows();
  if (k < 1 || k > N) throw ValidationError("k must be in [1, N]");
  if (policy.mode == CapacityMode::local_proportional && c_hat == nullptr)
    throw ValidationError("local_proportional capacity requires a target pattern");
  for (const Matrix& m : probs_per_process)
    if (m.cols() != N || m.rows() != S) throw ValidationError("per-process probability shapes differ");

  std::vector<RoutingResult> results(static_cast<size_t>(P));
  const size_t picks = static_cast<size_t>(P) * S * k, pn = static_cast<size_t>(P) * N;
  for (auto& res : results) {
    res.assignments.assign(static_cast<size_t>(S), std::vector<Assignment>(static_cast<size_t>(k)));
    res.counts.assign(static_cast<size_t>(N), 0);
    res.dropped.assign(static_cast<size_t>(N), 0);
    res.mean_probs.assign(static_cast<size_t>(N), 0.0);
  }
  if (S == 0) return results;

  std::vector<double> probs(static_cast<size_t>(P) * S * N);
  for (int i = 0; i < P; ++i)
    std::memcpy(probs.data() + static_cast<size_t>(i) * S * N, probs_per_process[static_cast<size_t>(i)].data().data(),
                sizeof(double) * S * N);
  std::vector<double> ch;
  if (c_hat != nullptr && policy.mode == CapacityMode::local_proportional) {
    if (c_hat->rows() != P || c_hat->cols() != N) throw ValidationError("target pattern must be P x N");
    ch = c_hat->data();
  }
  std::vector<long long> caps(pn);
  check(tamoe_capacity_caps(cap_mode(policy.mode), policy.capacity_factor, k, S, N, P, ch.empty() ? nullptr : ch.data(),
                            caps.data()));

  Router& router = router_for(P, S, N, k);
  const double* dprobs = upload(kP, probs.data(), probs.size());
  check(tamoe_router_route_probs(router.r, dprobs, cap_mode(policy.mode), caps.data(), nullptr));
  const auto idx = router.read<int>(TAMOE_R_IDX, picks);
  const auto gate = router.read<double>(TAMOE_R_GATE64, picks);
  const auto score = router.read<double>(TAMOE_R_SCORE, picks);
  const auto kept = router.read<unsigned char>(TAMOE_R_KEPT, picks);
  const auto counts = router.read<int>(TAMOE_R_COUNTS, pn);
  const auto dropped = router.read<int>(TAMOE_R_DROPPED, pn);
  const auto mean = router.read<double>(TAMOE_R_MEAN_PROBS, pn);

  for (int i = 0; i < P; ++i) {
    RoutingResult& res = results[static_cast<size_t>(i)];
    for (int s = 0; s < S; ++s)
      for (int slot = 0; slot < k; ++slot) {
        const size_t a = (static_cast<size_t>(i) * S + s) * k + slot;
        Assignment& as = res.assignments[static_cast<size_t>(s)][static_cast<size_t>(slot)];
        as.expert = idx[a];
        as.gate_value = gate[a];
        as.score = score[a];
        as.kept = kept[a] != 0;
      }
    for (int e = 0; e < N; ++e) {
      res.counts[static_cast<size_t>(e)] = counts[static_cast<size_t>(i) * N + e];
      res.dropped[static_cast<size_t>(e)] = dropped[static_cast<size_t>(i) * N + e];
      res.mean_probs[static_cast<size_t>(e)] = mean[static_cast<size_t>(i) * N + e];
    }
  }
  return results;
}

RoutingResult topk_route(const Matrix& probs, int k, const CapacityPolicy& policy, const Matrix* c_hat) {
  return topk_route(std::vector<Matrix>{probs}, k, policy, c_hat)[0];
}

std::vector<long long> largest_remainder_round(std::span<const double> values, long long target) {
  std::vector<long long> out(values.size());
  if (values.empty()) return out;
  check(tamoe_largest_remainder_round(values.data(), static_cast<int>(values.size()), target, out.data()));
  return out;
}

double loss_balance(const RoutingResult& result, int S) {
  double loss = 0.0;
  check(tamoe_loss_balance(result.counts.data(), result.mean_probs.data(), static_cast<int>(result.counts.size()), S,
                           &loss));
  return loss;
}

PenaltyNorm penalty_norm_from_string(const std::string& s) {
  if (s == "sum" || s == "sum_norm") return PenaltyNorm::sum_norm;
  if (s == "softmax") return PenaltyNorm::softmax;
  throw ValidationError("unknown penalty normalization: " + s);
}

std::vector<double> penalty_weights(std::span<const double> c_hat_row, PenaltyNorm norm, double temperature) {
  std::vector<double> p(c_hat_row.size());
  if (c_hat_row.empty()) return p;
  check(tamoe_penalty_weights(c_hat_row.data(), static_cast<int>(c_hat_row.size()),
                              norm == PenaltyNorm::sum_norm ? TAMOE_NORM_SUM : TAMOE_NORM_SOFTMAX, temperature,
                              p.data()));
  return p;
}

double loss_topo(const RoutingResult& result, std::span<const double> penalty, int N, int P, int S) {
  if (penalty.size() != result.counts.size()) throw ValidationError("penalty row size does not match expert count");
  double loss = 0.0;
  check(tamoe_loss_topo(result.counts.data(), result.mean_probs.data(), penalty.data(),
                        static_cast<int>(result.counts.size()), N, P, S, &loss));
  return loss;
}

Matrix grad_aux_loss(const Matrix& x, const Matrix& probs, std::span<const double> coeff) {
  const int S = probs.rows(), N = probs.cols(), d = x.cols();
  if (x.rows() != S) throw ValidationError("grad_aux_loss: x and probs need the same rows");
  if (coeff.size() != static_cast<size_t>(N)) throw ValidationError("grad_aux_loss: one coefficient per expert");
  Matrix grad(d, N);
  if (grad.data().empty()) return grad;
  const double* dx = upload(kX, x.data().data(), x.data().size());
  const double* dp = upload(kP, probs.data().data(), probs.data().size());
  double* dg = scratch().get<double>(kG, grad.data().size());
  check(tamoe_grad_aux_loss_f64(dx, dp, coeff.data(), S, d, N, dg, nullptr));
  download(grad.data().data(), dg, grad.data().size());
  return grad;
}

std::vector<double> balance_coefficients(const RoutingResult& result, int S) {
  std::vector<double> coeff(result.counts.size());
  check(tamoe_aux_coefficients(TAMOE_LOSS_BALANCE, result.counts.data(), nullptr, static_cast<int>(coeff.size()), 0,
                               0, S, coeff.data()));
  return coeff;
}

std::vector<double> topo_coefficients(const RoutingResult& result, std::span<const double> penalty, int N, int P,
                                      int S) {
  std::vector<double> coeff(result.counts.size());
  if (penalty.size() < coeff.size()) throw ValidationError("penalty row size does not match expert count");
  check(tamoe_aux_coefficients(TAMOE_LOSS_TOPO, result.counts.data(), penalty.data(), static_cast<int>(coeff.size()),
                               N, P, S, coeff.data()));
  return coeff;
}

Matrix grad_loss_balance(const Matrix& x, const Matrix& probs, const RoutingResult& result, int S) {
  return grad_aux_loss(x, probs, balance_coefficients(result, S));
}

Matrix grad_loss_topo(const Matrix& x, const Matrix& probs, const RoutingResult& result,
                      std::span<const double> penalty, int N, int P, int S) {
  return grad_aux_loss(x, probs, topo_coefficients(result, penalty, N, P, S));
}

}  // namespace tad
