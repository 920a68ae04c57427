// Host-side, once-per-topology inputs of the TA-MoE hot path: the closed-form
// dispatch target c_hat (Eq. 8), the penalty weights p = Norm(1/c_hat), and the
// per-(process, expert) capacities derived from them.  fp64, same arithmetic
// order as the reference so results are bit-identical.
#include "host_topology.hpp"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>

#include "common.hpp"

namespace tamoe {

// gate.cpp:52-78: floor(v + 1e-9), hand out the leftover by largest remainder
// (ties -> lower index), trim from the smallest remainders if over target.
std::vector<long long> largest_remainder_round(const double* values, int n, long long target) {
  std::vector<long long> out(static_cast<size_t>(n), 0);
  std::vector<int> order(static_cast<size_t>(n));
  std::vector<double> rem(static_cast<size_t>(n));
  long long assigned = 0;
  for (int i = 0; i < n; ++i) {
    const double v = values[i] > 0.0 ? values[i] : 0.0;
    out[i] = static_cast<long long>(std::floor(v + 1e-9));
    assigned += out[i];
    rem[i] = v - static_cast<double>(out[i]);
  }
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return rem[a] != rem[b] ? rem[a] > rem[b] : a < b; });
  long long left = target - assigned;
  for (int r = 0; r < n && left > 0; ++r, --left) out[order[r]] += 1;
  for (int r = n - 1; r >= 0 && left < 0; --r) {
    if (out[order[r]] > 0) {
      out[order[r]] -= 1;
      ++left;
    }
  }
  return out;
}

// gate.cpp:222-246
std::vector<double> penalty_weights(const double* c_hat_row, int n, int norm, double temperature) {
  std::vector<double> inv(static_cast<size_t>(n)), p(static_cast<size_t>(n));
  for (int e = 0; e < n; ++e) {
    require(c_hat_row[e] > 0.0, "penalty weights need strictly positive targets");
    inv[e] = 1.0 / c_hat_row[e];
  }
  if (norm == 0) {
    double total = 0.0;
    for (double v : inv) total += v;
    for (int e = 0; e < n; ++e) p[e] = inv[e] / total;
  } else {
    double t = temperature;
    if (!(t > 0.0)) {
      double s = 0.0;
      for (double v : inv) s += v;
      t = s / static_cast<double>(n);
    }
    double zmax = -std::numeric_limits<double>::infinity();
    for (double v : inv) zmax = std::max(zmax, v / t);
    double denom = 0.0;
    for (int e = 0; e < n; ++e) {
      p[e] = std::exp(inv[e] / t - zmax);
      denom += p[e];
    }
    for (double& v : p) v /= denom;
  }
  return p;
}

// solver.cpp:28-52, Eq. 8: c_ie = kS / (E * sum_j(1/beta_ij) * beta_{i, dev(e)})
std::vector<double> target_closed_form(const double* beta, int P, int N, int k, int S) {
  require(k >= 1 && S >= 1 && N >= 1 && P >= 1, "k, S, N, P must be positive");
  require(N % P == 0, "N must be divisible by P");
  require(k <= N, "k cannot exceed N");
  for (int i = 0; i < P * P; ++i) require(beta[i] > 0.0, "closed form requires strictly positive beta_hat");
  const int E = N / P;
  const double row_target = static_cast<double>(k) * S;
  std::vector<double> c(static_cast<size_t>(P) * N);
  for (int i = 0; i < P; ++i) {
    double inv_sum = 0.0;
    for (int j = 0; j < P; ++j) inv_sum += 1.0 / beta[i * P + j];
    for (int e = 0; e < N; ++e) c[static_cast<size_t>(i) * N + e] = row_target / (E * inv_sum * beta[i * P + e / E]);
  }
  return c;
}

// gate.cpp:151-180 (cap per capacity domain) laid out per (process, expert).
std::vector<long long> capacity_caps(int mode, double cf, int k, int S, int N, int P, const double* c_hat) {
  require(k >= 1 && k <= N, "k must be in [1, N]");
  std::vector<long long> caps(static_cast<size_t>(P) * N, std::numeric_limits<long long>::max());
  if (mode == 0) return caps;
  const double cap_real = cf * static_cast<double>(k) * S * P / N;  // gate.hpp:46-48
  if (mode == 1) {
    const long long c = static_cast<long long>(std::floor(cap_real + 1e-9));
    std::fill(caps.begin(), caps.end(), c);
  } else if (mode == 2) {
    const long long c = static_cast<long long>(std::floor(cap_real / P + 1e-9));
    std::fill(caps.begin(), caps.end(), c);
  } else if (mode == 3) {
    require(c_hat != nullptr, "local_proportional capacity requires a target pattern");
    std::vector<double> w(static_cast<size_t>(P));
    for (int e = 0; e < N; ++e) {
      double col = 0.0;
      for (int i = 0; i < P; ++i) {
        w[i] = c_hat[static_cast<size_t>(i) * N + e];
        col += w[i];
      }
      require(col > 0.0, "target pattern column sums to zero");
      for (double& v : w) v *= cap_real / col;
      auto r = largest_remainder_round(w.data(), P, static_cast<long long>(std::floor(cap_real + 1e-9)));
      for (int i = 0; i < P; ++i) caps[static_cast<size_t>(i) * N + e] = r[i];
    }
  } else {
    throw ValidationError("unknown capacity mode");
  }
  return caps;
}

// dispatch.cpp:21-26
std::vector<double> device_payload_tokens(const double* counts, int P, int N) {
  require(P >= 1 && N % P == 0, "N must be divisible by P");
  const int E = N / P;
  std::vector<double> out(static_cast<size_t>(P) * P, 0.0);
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) {
      double t = 0.0;
      for (int e = j * E; e < (j + 1) * E; ++e) t += counts[static_cast<size_t>(i) * N + e];
      out[static_cast<size_t>(i) * P + j] = t;
    }
  return out;
}

// gate.cpp:209-214: sum_e m_e * (c_e / S), expert order
double loss_balance(const long long* counts, const double* mean_probs, int N, int S) {
  double loss = 0.0;
  for (int e = 0; e < N; ++e) loss += mean_probs[e] * (static_cast<double>(counts[e]) / S);
  return loss;
}

// gate.cpp:248-255: N * P * sum_e p_e * m_e * (c_e / S)
double loss_topo(const long long* counts, const double* mean_probs, const double* penalty, int n, int N, int P, int S) {
  double loss = 0.0;
  for (int e = 0; e < n; ++e) loss += penalty[e] * mean_probs[e] * (static_cast<double>(counts[e]) / S);
  return static_cast<double>(N) * P * loss;
}

// gate.cpp:273-287: balance c_e / S^2; topo N*P/S^2 * p_e * c_e
std::vector<double> aux_coefficients(int kind, const long long* counts, const double* penalty, int n, int N, int P,
                                     int S) {
  std::vector<double> coeff(static_cast<size_t>(n));
  if (kind == 0) {
    const double s2 = static_cast<double>(S) * S;
    for (int e = 0; e < n; ++e) coeff[e] = static_cast<double>(counts[e]) / s2;
  } else {
    require(penalty != nullptr, "topo coefficients need the penalty row");
    const double scale = static_cast<double>(N) * P / (static_cast<double>(S) * S);
    for (int e = 0; e < n; ++e) coeff[e] = scale * penalty[e] * static_cast<double>(counts[e]);
  }
  return coeff;
}

}  // namespace tamoe
