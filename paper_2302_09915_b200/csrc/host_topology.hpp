#pragma once
#include <vector>

namespace tamoe {

std::vector<long long> largest_remainder_round(const double* values, int n, long long target);
std::vector<double> penalty_weights(const double* c_hat_row, int n, int norm, double temperature);
std::vector<double> target_closed_form(const double* beta, int P, int N, int k, int S);
std::vector<long long> capacity_caps(int mode, double cf, int k, int S, int N, int P, const double* c_hat);
std::vector<double> device_payload_tokens(const double* counts, int P, int N);
// Auxiliary losses / gradient coefficients on a routing result (gate.cpp:209-214, 248-255, 273-287).
double loss_balance(const long long* counts, const double* mean_probs, int N, int S);
double loss_topo(const long long* counts, const double* mean_probs, const double* penalty, int n, int N, int P, int S);
std::vector<double> aux_coefficients(int kind, const long long* counts, const double* penalty, int n, int N, int P,
                                     int S);

// ---- measured-topology pipeline (host_profile.cpp)
std::vector<int> check_tree_levels(const int* levels, int n_levels, int P);
std::vector<std::vector<int>> device_groups(const std::vector<int>& levels, int device);
void fit_profile(const int* src, const int* dst, const double* mb, const double* us, int n, int P, double* alpha,
                 double* beta);
void fill_partial_profile(const double* alpha, const double* beta, int P, const int* levels, int n_levels,
                          double self_beta_floor, double* alpha_out, double* beta_out);
void smooth_profile(const int* levels, int n_levels, const double* alpha, const double* beta, int P,
                    double self_beta_floor, double* alpha_hat, double* beta_hat, std::vector<double>* level_alpha,
                    std::vector<double>* level_beta);
struct ExchangeCost {
  std::vector<double> pair_cost_us, per_device_send_us, per_device_recv_us;
  double bottleneck_us = 0.0, total_bytes = 0.0, size_exchange_us = 0.0, total_estimate_us = 0.0;
};
ExchangeCost exchange_cost(const double* alpha, const double* beta, const double* c, int P, int N, int d, int b,
                           int extra_alpha_rounds);

}  // namespace tamoe
