// extern "C" boundary (include/tamoe.h).  Each entry point translates C++
// exceptions into the reference's status convention via guarded().
#include "../../include/tamoe.h"

#include <cstring>

#include "capi_util.hpp"
#include "expert.hpp"
#include "host_topology.hpp"

using namespace tamoe;

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

}  // extern "C"
