// Measured-topology pipeline, host side: per-link alpha/beta fitted from timed
// transfers, completion of partially measured profiles, level smoothing over a symmetric switch tree
// and the alpha-beta exchange-cost model.  fp64 and the reference's accumulation orders, so the results
// match the reference bit for bit (tests/test_profile.py against oracle/_ref).
//
// Trees are given by their level vector, root first (`[8]` = one switch, `[2,4]` = two groups of four):
// the symmetric trees the reference smooths over (topology.hpp:28-33).
#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "common.hpp"
#include "host_topology.hpp"

namespace tamoe {

namespace {

constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();
bool missing(double v) { return std::isnan(v); }

// Leaf index -> digits of the subtree it sits in at every switch level (mixed radix over the levels).
std::vector<int> tree_path(const std::vector<int>& levels, int device) {
  const int L = static_cast<int>(levels.size());
  // devices under one switch of depth l (the root is depth 0, leaf-group switches depth L - 1)
  std::vector<int> below(static_cast<size_t>(L), 1);
  below[static_cast<size_t>(L) - 1] = levels[static_cast<size_t>(L) - 1];
  for (int l = L - 2; l >= 0; --l) below[static_cast<size_t>(l)] = below[static_cast<size_t>(l) + 1] * levels[static_cast<size_t>(l)];
  // the switch at depth l that the device hangs under is identified by device / below[l]
  std::vector<int> path(static_cast<size_t>(L));
  for (int l = 0; l < L; ++l) path[static_cast<size_t>(l)] = device / below[static_cast<size_t>(l)];
  return path;
}

int tree_devices(const std::vector<int>& levels) {
  int p = 1;
  for (int v : levels) p *= v;
  return p;
}

double mean_present(const std::vector<double>& m, int P, const std::vector<std::pair<int, int>>& pairs) {
  double sum = 0.0;
  long long n = 0;
  for (auto [i, j] : pairs) {
    const double v = m[static_cast<size_t>(i) * P + j];
    if (missing(v)) continue;
    sum += v;
    ++n;
  }
  return n ? sum / static_cast<double>(n) : kNaN;
}

void validate_profile(const std::vector<double>& alpha, const std::vector<double>& beta, int P, double floor) {
  if (!(floor > 0.0)) throw ValidationError("self_beta_floor must be positive");
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) {
      const double a = alpha[static_cast<size_t>(i) * P + j], b = beta[static_cast<size_t>(i) * P + j];
      if (!(a >= 0.0) || !(b >= 0.0)) throw ValidationError("profile entries must be finite and nonnegative");
      if (i == j && b < floor) throw ValidationError("diagonal beta below self_beta_floor");
    }
}

}  // namespace

std::vector<int> check_tree_levels(const int* levels, int n_levels, int P) {
  require(n_levels >= 1 && levels != nullptr, "tree topology needs at least one level");
  std::vector<int> lv(levels, levels + n_levels);
  for (int v : lv) require(v >= 1, "tree group sizes must be positive");
  require(tree_devices(lv) == P, "tree levels do not multiply to the device count");
  return lv;
}

// topology.cpp:258-287: devices grouped by the number of switches crossed on the way from `device`
// (up to the lowest common switch, across it, down); group 0 also holds the device itself, sorted.
std::vector<std::vector<int>> device_groups(const std::vector<int>& levels, int device) {
  const int P = tree_devices(levels);
  require(device >= 0 && device < P, "device index out of range");
  const std::vector<int> pi = tree_path(levels, device);
  const int L = static_cast<int>(levels.size());
  std::map<int, std::vector<int>> by_count;
  for (int j = 0; j < P; ++j) {
    if (j == device) continue;
    const std::vector<int> pj = tree_path(levels, j);
    int common = 0;
    while (common < L && pi[static_cast<size_t>(common)] == pj[static_cast<size_t>(common)]) ++common;
    by_count[2 * (L - common) + 1].push_back(j);
  }
  std::vector<std::vector<int>> groups;
  for (auto& kv : by_count) groups.push_back(std::move(kv.second));
  if (groups.empty()) groups.emplace_back();
  groups[0].push_back(device);
  std::sort(groups[0].begin(), groups[0].end());
  return groups;
}

// comm_cost.cpp:57-104: per ordered pair, least squares time = alpha + beta * MB over its samples (in
// sample order); one message size -> alpha = 0, beta = mean(time / size); alpha < 0 -> refit through the
// origin.  Unobserved pairs stay NaN.
void fit_profile(const int* src, const int* dst, const double* mb, const double* us, int n, int P, double* alpha,
                 double* beta) {
  if (n <= 0) throw ValidationError("fit_profile needs at least one sample");
  require(P >= 1, "device count must be positive");
  std::map<std::pair<int, int>, std::vector<int>> by_pair;
  for (int s = 0; s < n; ++s) {
    if (src[s] < 0 || dst[s] < 0) throw ValidationError("negative device index in samples");
    if (!(mb[s] > 0.0)) throw ValidationError("message sizes must be positive");
    if (src[s] >= P || dst[s] >= P) throw ValidationError("sample device index >= device count");
    by_pair[{src[s], dst[s]}].push_back(s);
  }
  for (int i = 0; i < P * P; ++i) alpha[i] = beta[i] = kNaN;
  for (const auto& [pair, group] : by_pair) {
    double lo = mb[group[0]], hi = mb[group[0]];
    for (int s : group) {
      lo = std::min(lo, mb[s]);
      hi = std::max(hi, mb[s]);
    }
    double a = 0.0, b = 0.0;
    if (hi - lo < 1e-12 * hi) {
      for (int s : group) b += us[s] / mb[s];
      b /= static_cast<double>(group.size());
    } else {
      double sx = 0.0, sy = 0.0, sxx = 0.0, sxy = 0.0;
      const double cnt = static_cast<double>(group.size());
      for (int s : group) {
        sx += mb[s];
        sy += us[s];
        sxx += mb[s] * mb[s];
        sxy += mb[s] * us[s];
      }
      b = (cnt * sxy - sx * sy) / (cnt * sxx - sx * sx);
      a = (sy - b * sx) / cnt;
      if (a < 0.0) {
        a = 0.0;
        b = sxy / sxx;
      }
    }
    if (!(b > 0.0))
      throw ValidationError("fitted beta is not positive for pair " + std::to_string(pair.first) + "->" +
                            std::to_string(pair.second));
    alpha[pair.first * P + pair.second] = a;
    beta[pair.first * P + pair.second] = b;
  }
}

// profile.cpp:164-233: (1) symmetry, (2) per-level mean over the tree (when given), then the global
// off-diagonal mean, (3) diagonal from the measured self links, else min off-diagonal beta / 10, clamped.
void fill_partial_profile(const double* alpha_in, const double* beta_in, int P, const int* levels, int n_levels,
                          double floor, double* alpha_out, double* beta_out) {
  require(P >= 1, "device count must be positive");
  std::vector<double> A(alpha_in, alpha_in + static_cast<size_t>(P) * P), B(beta_in, beta_in + static_cast<size_t>(P) * P);
  std::vector<std::vector<std::vector<int>>> groups;
  if (n_levels > 0) {
    const std::vector<int> lv = check_tree_levels(levels, n_levels, P);
    for (int i = 0; i < P; ++i) groups.push_back(device_groups(lv, i));
  }
  std::vector<std::pair<int, int>> offdiag;
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j)
      if (i != j) offdiag.emplace_back(i, j);
  for (std::vector<double>* m : {&A, &B}) {
    auto at = [&](int i, int j) -> double& { return (*m)[static_cast<size_t>(i) * P + j]; };
    for (int i = 0; i < P; ++i)
      for (int j = 0; j < P; ++j)
        if (missing(at(i, j)) && !missing(at(j, i))) at(i, j) = at(j, i);
    if (!groups.empty()) {
      for (size_t l = 0; l < groups[0].size(); ++l) {
        std::vector<std::pair<int, int>> lp;
        for (int i = 0; i < P; ++i)
          for (int j : groups[static_cast<size_t>(i)][l])
            if (j != i) lp.emplace_back(i, j);
        const double avg = mean_present(*m, P, lp);
        for (auto [i, j] : lp)
          if (missing(at(i, j)) && !missing(avg)) at(i, j) = avg;
      }
    }
    const double gavg = mean_present(*m, P, offdiag);
    for (auto [i, j] : offdiag)
      if (missing(at(i, j))) {
        if (missing(gavg)) throw ValidationError("profile has no measured off-diagonal entries");
        at(i, j) = gavg;
      }
  }
  std::vector<std::pair<int, int>> diag;
  for (int i = 0; i < P; ++i) diag.emplace_back(i, i);
  const double da = mean_present(A, P, diag), db = mean_present(B, P, diag);
  double min_off = std::numeric_limits<double>::infinity();
  for (auto [i, j] : offdiag) min_off = std::min(min_off, B[static_cast<size_t>(i) * P + j]);
  for (int i = 0; i < P; ++i) {
    double& a = A[static_cast<size_t>(i) * P + i];
    double& b = B[static_cast<size_t>(i) * P + i];
    if (missing(a)) a = missing(da) ? 0.0 : da;
    if (missing(b)) b = missing(db) ? min_off / 10.0 : db;
    b = std::max(b, floor);
  }
  validate_profile(A, B, P, floor);
  std::copy(A.begin(), A.end(), alpha_out);
  std::copy(B.begin(), B.end(), beta_out);
}

// profile.cpp:46-98: every link of a level shares the plain mean over all ordered pairs of that level;
// the diagonal is the mean measured self cost (beta clamped at the floor).
void smooth_profile(const int* levels, int n_levels, const double* alpha, const double* beta, int P, double floor,
                    double* alpha_hat, double* beta_hat, std::vector<double>* level_alpha,
                    std::vector<double>* level_beta) {
  const std::vector<int> lv = check_tree_levels(levels, n_levels, P);
  std::vector<double> A(alpha, alpha + static_cast<size_t>(P) * P), B(beta, beta + static_cast<size_t>(P) * P);
  validate_profile(A, B, P, floor);
  std::vector<std::vector<std::vector<int>>> groups;
  for (int i = 0; i < P; ++i) groups.push_back(device_groups(lv, i));
  const size_t L = groups[0].size();
  std::vector<double> la(L, 0.0), lb(L, 0.0);
  std::vector<long long> cnt(L, 0);
  for (int i = 0; i < P; ++i)
    for (size_t l = 0; l < L; ++l)
      for (int j : groups[static_cast<size_t>(i)][l]) {
        if (j == i) continue;
        la[l] += A[static_cast<size_t>(i) * P + j];
        lb[l] += B[static_cast<size_t>(i) * P + j];
        ++cnt[l];
      }
  for (size_t l = 0; l < L; ++l) {
    if (cnt[l] == 0) {
      if (l == 0 && lv.back() == 1) continue;
      throw ValidationError("empty level group while smoothing");
    }
    la[l] /= static_cast<double>(cnt[l]);
    lb[l] /= static_cast<double>(cnt[l]);
  }
  double da = 0.0, db = 0.0;
  for (int i = 0; i < P; ++i) {
    da += A[static_cast<size_t>(i) * P + i];
    db += B[static_cast<size_t>(i) * P + i];
  }
  da /= P;
  db = std::max(db / P, floor);
  for (int i = 0; i < P; ++i) {
    alpha_hat[static_cast<size_t>(i) * P + i] = da;
    beta_hat[static_cast<size_t>(i) * P + i] = db;
    for (size_t l = 0; l < L; ++l)
      for (int j : groups[static_cast<size_t>(i)][l]) {
        if (j == i) continue;
        alpha_hat[static_cast<size_t>(i) * P + j] = la[l];
        beta_hat[static_cast<size_t>(i) * P + j] = lb[l];
      }
  }
  if (level_alpha) *level_alpha = la;
  if (level_beta) *level_beta = lb;
}

// comm_cost.cpp:15-55: pair cost alpha_ij + beta_ij * (tokens i sends to device j) * d * b / 1e6 MB;
// the exchange is bounded by its slowest delivery, plus optional latency-only rounds (max alpha each).
ExchangeCost exchange_cost(const double* alpha, const double* beta, const double* c, int P, int N, int d, int b,
                           int extra_alpha_rounds) {
  require(P >= 1 && N >= P && N % P == 0, "N must be a positive multiple of P");
  require(d >= 1 && b >= 1, "d and bytes per element must be positive");
  for (long long i = 0; i < static_cast<long long>(P) * N; ++i)
    if (!(c[i] >= 0.0) || !std::isfinite(c[i])) throw ValidationError("dispatch matrix entries must be finite and >= 0");
  const std::vector<double> payload = device_payload_tokens(c, P, N);
  const double mb_per_token = static_cast<double>(d) * b / 1e6;
  ExchangeCost r;
  r.pair_cost_us.assign(static_cast<size_t>(P) * P, 0.0);
  r.per_device_send_us.assign(static_cast<size_t>(P), 0.0);
  r.per_device_recv_us.assign(static_cast<size_t>(P), 0.0);
  double max_alpha = 0.0;
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) {
      const size_t ij = static_cast<size_t>(i) * P + j;
      const double cost = alpha[ij] + beta[ij] * (payload[ij] * mb_per_token);
      if (!std::isfinite(cost)) throw ValidationError("pair cost overflows the representable range");
      r.pair_cost_us[ij] = cost;
      r.bottleneck_us = std::max(r.bottleneck_us, cost);
      r.per_device_send_us[static_cast<size_t>(i)] = std::max(r.per_device_send_us[static_cast<size_t>(i)], cost);
      r.per_device_recv_us[static_cast<size_t>(j)] = std::max(r.per_device_recv_us[static_cast<size_t>(j)], cost);
      max_alpha = std::max(max_alpha, alpha[ij]);
    }
  double tokens = 0.0;
  for (long long i = 0; i < static_cast<long long>(P) * N; ++i) tokens += c[i];
  r.total_bytes = tokens * d * b;
  r.size_exchange_us = extra_alpha_rounds * max_alpha;
  r.total_estimate_us = r.bottleneck_us + r.size_exchange_us;
  return r;
}

}  // namespace tamoe
