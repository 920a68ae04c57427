#pragma once
#include <vector>

namespace tamoe {

std::vector<long long> largest_remainder_round(const double* values, int n, long long target);
std::vector<double> penalty_weights(const double* c_hat_row, int n, int norm, double temperature);
std::vector<double> target_closed_form(const double* beta, int P, int N, int k, int S);
std::vector<long long> capacity_caps(int mode, double cf, int k, int S, int N, int P, const double* c_hat);
std::vector<double> device_payload_tokens(const double* counts, int P, int N);

}  // namespace tamoe
