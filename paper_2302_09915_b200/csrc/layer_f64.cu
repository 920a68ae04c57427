// Reference-precision (fp64) MoE layer step with linear experts: BASELINE config 1 on the device.
// See layer_f64.hpp.  Reference order followed per kernel (trainer.cpp):
//   expert fwd   :284-289  out[j] = sum over r ascending of x_r * U_e(r, j), skipping x_r == 0
//   combine      :279-296  y_hat[j] = sum over kept slots (slot order) of g * out[j]; residual = y_hat - y;
//                          task += residual^2
//   dL/dg        :298-308  dldg = (2 / (P S d_out)) * sum over j ascending of residual[j] * out[j]
//   expert grad  :310-316  dU_e(r, j) += ((mse_scale * g) * x_r) * residual[j] over (process, token) ascending
//   Jacobian     :318-331  top-1: dpi_e += dldg; top-k: sum_j dldg_j (delta_jl M - p_j) / M^2
//   aux          :334-345  loss_topo / loss_balance and their coefficients (gate.cpp:209-287), dpi += (w/P) coeff
//   softmax bwd  :347-355  dz = p (dpi - <dpi, p>), dW = x^T dz (add_atb, gate_f64.cu)
// Products and sums are separately rounded (__dmul_rn / __dadd_rn): the reference is built without FMA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.hpp"
#include "gate_f64.hpp"
#include "host_topology.hpp"
#include "layer_f64.hpp"

namespace tamoe {
namespace {

constexpr int kT = 16;

__device__ __forceinline__ int kept_rows(const RouteBuffers& b, int P, int N, int e) {
  int c = 0;
  for (int p = 0; p < P; ++p) c += b.counts[p * N + e];
  return c;
}

// out[pick][j] for the kept picks of expert blockIdx.z (clist order); grid (ceil(dout/16), ceil(rows/16), N)
__global__ void expert_fwd_f64_kernel(RouteDims dm, RouteBuffers b, const double* __restrict__ x,
                                      const double* __restrict__ U, int d, int dout, double* __restrict__ out) {
  __shared__ double xs[kT][kT + 1];
  __shared__ double us[kT][kT + 1];
  __shared__ int tok[kT], pick[kT];
  const int e = blockIdx.z;
  const int rows = kept_rows(b, dm.P, dm.N, e);
  const int r0 = blockIdx.y * kT;
  if (r0 >= rows) return;
  if (threadIdx.y == 0 && threadIdx.x < kT) {
    const int rr = r0 + threadIdx.x;
    const int pk = rr < rows ? b.clist[b.list_start[e] + rr] : -1;
    pick[threadIdx.x] = pk;
    tok[threadIdx.x] = pk >= 0 ? pk / dm.k : -1;
  }
  __syncthreads();
  const double* Ue = U + static_cast<long long>(e) * d * dout;
  const int j = blockIdx.x * kT + threadIdx.x;
  double acc = 0.0;
  for (int k0 = 0; k0 < d; k0 += kT) {
    {
      const int t = tok[threadIdx.y], kk = k0 + threadIdx.x;
      xs[threadIdx.y][threadIdx.x] = (t >= 0 && kk < d) ? x[static_cast<long long>(t) * d + kk] : 0.0;
      const int kr = k0 + threadIdx.y;
      us[threadIdx.y][threadIdx.x] = (kr < d && j < dout) ? Ue[static_cast<long long>(kr) * dout + j] : 0.0;
    }
    __syncthreads();
    const int kend = min(kT, d - k0);
    for (int kk = 0; kk < kend; ++kk) {
      const double xv = xs[threadIdx.y][kk];
      if (xv != 0.0) acc = __dadd_rn(acc, __dmul_rn(xv, us[kk][threadIdx.x]));
    }
    __syncthreads();
  }
  const int pk = pick[threadIdx.y];
  if (pk >= 0 && j < dout) out[static_cast<long long>(pk) * dout + j] = acc;
}

// One block per token: y_hat / residual (parallel over j, each element in slot order), then dL/dg per slot and
// the token's sum of squared residuals, each by one thread walking j in order.
__global__ void combine_f64_kernel(RouteDims dm, RouteBuffers b, const double* __restrict__ out,
                                   const double* __restrict__ y, int dout, double mse_scale,
                                   double* __restrict__ resid, double* __restrict__ y_hat, double* __restrict__ dldg,
                                   double* __restrict__ task_part) {
  extern __shared__ double rs[];  // [dout]
  const long long t = blockIdx.x;
  const int k = dm.k;
  for (int j = threadIdx.x; j < dout; j += blockDim.x) {
    double acc = 0.0;
    for (int sl = 0; sl < k; ++sl) {
      const long long a = t * k + sl;
      if (!b.kept[a]) continue;
      acc = __dadd_rn(acc, __dmul_rn(b.gate64[a], out[a * dout + j]));
    }
    if (y_hat) y_hat[t * dout + j] = acc;
    const double r = __dadd_rn(acc, -y[t * dout + j]);
    rs[j] = r;
    resid[t * dout + j] = r;
  }
  __syncthreads();
  if (threadIdx.x < k) {
    const long long a = t * k + threadIdx.x;
    double v = 0.0;
    if (b.kept[a]) {
      const double* o = out + a * dout;
      double dot = 0.0;
      for (int j = 0; j < dout; ++j) dot = __dadd_rn(dot, __dmul_rn(rs[j], o[j]));
      v = __dmul_rn(mse_scale, dot);
    }
    dldg[a] = v;
  } else if (threadIdx.x == k) {
    double sq = 0.0;
    for (int j = 0; j < dout; ++j) sq = __dadd_rn(sq, __dmul_rn(rs[j], rs[j]));
    task_part[t] = sq;
  }
}

// dU_e(r, j) over the kept picks of expert blockIdx.z in clist ((process, token)) order;
// grid (ceil(dout/16), ceil(d/16), N)
__global__ void expert_wgrad_f64_kernel(RouteDims dm, RouteBuffers b, const double* __restrict__ x,
                                        const double* __restrict__ resid, int d, int dout, double mse_scale,
                                        double* __restrict__ dU) {
  __shared__ double as[kT][kT + 1];  // [row][r]
  __shared__ double rsd[kT][kT + 1];  // [row][j]
  __shared__ int tok[kT];
  __shared__ double gsc[kT];
  const int e = blockIdx.z;
  const int rows = kept_rows(b, dm.P, dm.N, e);
  const int r = blockIdx.y * kT + threadIdx.y;
  const int j = blockIdx.x * kT + threadIdx.x;
  double acc = 0.0;
  for (int q0 = 0; q0 < rows; q0 += kT) {
    if (threadIdx.y == 0 && threadIdx.x < kT) {
      const int q = q0 + threadIdx.x;
      const int pk = q < rows ? b.clist[b.list_start[e] + q] : -1;
      tok[threadIdx.x] = pk >= 0 ? pk / dm.k : -1;
      gsc[threadIdx.x] = pk >= 0 ? __dmul_rn(mse_scale, b.gate64[pk]) : 0.0;
    }
    __syncthreads();
    {
      // as[row][c] = (mse_scale * g_row) * x[tok_row][blockIdx.y*16 + c]; rsd[row][c] = resid[tok_row][j0 + c]
      const int row = threadIdx.y, c = threadIdx.x;
      const int t = tok[row];
      const int rc = blockIdx.y * kT + c, jc = blockIdx.x * kT + c;
      as[row][c] = (t >= 0 && rc < d) ? __dmul_rn(gsc[row], x[static_cast<long long>(t) * d + rc]) : 0.0;
      rsd[row][c] = (t >= 0 && jc < dout) ? resid[static_cast<long long>(t) * dout + jc] : 0.0;
    }
    __syncthreads();
    const int qend = min(kT, rows - q0);
    for (int q = 0; q < qend; ++q) {
      const double av = as[q][threadIdx.y];
      if (av != 0.0) acc = __dadd_rn(acc, __dmul_rn(av, rsd[q][threadIdx.x]));
    }
    __syncthreads();
  }
  if (r < d && j < dout) dU[(static_cast<long long>(e) * d + r) * dout + j] = acc;
}

// One block: mean probabilities (sequential over tokens, gate.cpp:115), per-process aux loss and coefficients
// (gate.cpp:209-214, 248-255, 273-287), step_aux / P and the task loss (trainer.cpp:359-360).
__global__ void aux_f64_kernel(RouteDims dm, RouteBuffers b, const double* __restrict__ probs,
                               const double* __restrict__ penalty, int kind, const double* __restrict__ task_part,
                               double task_den, double* __restrict__ mean, double* __restrict__ coeff,
                               double* __restrict__ losses) {
  const int P = dm.P, S = dm.S, N = dm.N;
  for (int pe = threadIdx.x; pe < P * N; pe += blockDim.x) {
    const int i = pe / N, e = pe % N;
    const double* p = probs + static_cast<long long>(i) * S * N + e;
    double m = 0.0;
    for (int s = 0; s < S; ++s) m = __dadd_rn(m, __ddiv_rn(p[static_cast<long long>(s) * N], static_cast<double>(S)));
    mean[pe] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double Sd = static_cast<double>(S);
    const double s2 = __dmul_rn(Sd, Sd);
    const double np = __dmul_rn(static_cast<double>(N), static_cast<double>(P));
    const double scale = __ddiv_rn(np, s2);
    double step_aux = 0.0;
    for (int i = 0; i < P; ++i) {
      double loss = 0.0;
      for (int e = 0; e < N; ++e) {
        const double c = static_cast<double>(b.counts[i * N + e]);
        const double m = mean[i * N + e];
        if (kind == 1) {
          loss = __dadd_rn(loss, __dmul_rn(__dmul_rn(penalty[i * N + e], m), __ddiv_rn(c, Sd)));
          coeff[i * N + e] = __dmul_rn(__dmul_rn(scale, penalty[i * N + e]), c);
        } else {
          loss = __dadd_rn(loss, __dmul_rn(m, __ddiv_rn(c, Sd)));
          coeff[i * N + e] = __ddiv_rn(c, s2);
        }
      }
      if (kind == 1) loss = __dmul_rn(np, loss);
      step_aux = __dadd_rn(step_aux, loss);
    }
    double task = 0.0;
    for (long long t = 0; t < static_cast<long long>(P) * S; ++t) task = __dadd_rn(task, task_part[t]);
    losses[0] = __ddiv_rn(task, task_den);
    losses[1] = __ddiv_rn(step_aux, static_cast<double>(P));
  }
}

// One thread per token: dpi (Jacobian of the kept gate values + aux term), then dz = p (dpi - <dpi, p>).
__global__ void gate_dz_f64_kernel(RouteDims dm, RouteBuffers b, const double* __restrict__ probs,
                                   const double* __restrict__ dldg, const double* __restrict__ coeff,
                                   double aux_scale, double* __restrict__ dz) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(dm.P) * dm.S) return;
  const int N = dm.N, k = dm.k;
  const int i = static_cast<int>(t / dm.S);
  const double* p = probs + t * N;
  double* g = dz + t * N;
  for (int e = 0; e < N; ++e) g[e] = 0.0;
  const long long a0 = t * k;
  if (k == 1) {
    if (b.kept[a0]) g[b.idx[a0]] = __dadd_rn(g[b.idx[a0]], dldg[a0]);
  } else {
    double mass = 0.0;
    for (int j = 0; j < k; ++j) mass = __dadd_rn(mass, b.score[a0 + j]);
    const double m2 = __dmul_rn(mass, mass);
    for (int l = 0; l < k; ++l) {
      double acc = 0.0;
      for (int j = 0; j < k; ++j) {
        const double dj = dldg[a0 + j];
        if (dj == 0.0) continue;
        const double del = j == l ? mass : 0.0;
        acc = __dadd_rn(acc, __ddiv_rn(__dmul_rn(dj, __dadd_rn(del, -b.score[a0 + j])), m2));
      }
      const int el = b.idx[a0 + l];
      g[el] = __dadd_rn(g[el], acc);
    }
  }
  for (int e = 0; e < N; ++e) g[e] = __dadd_rn(g[e], __dmul_rn(aux_scale, coeff[i * N + e]));
  double dot = 0.0;
  for (int e = 0; e < N; ++e) dot = __dadd_rn(dot, __dmul_rn(g[e], p[e]));
  for (int e = 0; e < N; ++e) g[e] = __dmul_rn(p[e], __dadd_rn(g[e], -dot));
}

template <class T>
struct Scratch {
  T* p = nullptr;
  cudaStream_t s;
  Scratch(long long n, cudaStream_t st) : s(st) {
    TAMOE_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * (n > 0 ? n : 1), s));
  }
  ~Scratch() { cudaFreeAsync(p, s); }
};

}  // namespace

void layer_step_f64(RouteWorkspace& rw, const F64StepArgs& a, cudaStream_t s) {
  const RouteDims& dm = rw.dims;
  const int P = dm.P, S = dm.S, N = dm.N, d = a.d, dout = a.d_out;
  require(d > 0 && dout > 0, "layer_step_f64: d and d_out must be positive");
  require(a.aux_kind >= 0 && a.aux_kind <= 2, "layer_step_f64: aux kind must be balance, topo or compulsory");
  require(a.aux_kind != 1 || a.penalty != nullptr, "layer_step_f64: topo loss needs penalty weights");
  require(a.aux_kind != 2 || (a.c_hat != nullptr && dm.k == 1),
          "compulsory routing supports top-1 only and requires a target pattern");
  require(a.x && a.y && a.gates && a.experts && a.gate_grads && a.expert_grads && a.losses && a.caps,
          "layer_step_f64: null buffer");
  require(rw.buf.gate64 != nullptr, "layer_step_f64: router without fp64 gate values");
  const long long T = static_cast<long long>(P) * S, picks = dm.picks();

  Scratch<double> probs_s(a.probs ? 0 : T * N, s);
  double* probs = a.probs ? a.probs : probs_s.p;
  Scratch<int> bad(1, s);
  TAMOE_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
  // gate_forward per process (trainer.cpp:247): bit-identical matmul, reference-order softmax
  for (int i = 0; i < P; ++i) {
    double* pi = probs + static_cast<long long>(i) * S * N;
    matmul_f64(a.x + static_cast<long long>(i) * S * d, a.gates + static_cast<long long>(i) * d * N, pi, S, N, d, s);
    softmax_rows_f64(pi, pi, S, N, bad.p, s);
  }
  int bad_h = 0;
  TAMOE_CUDA(cudaMemcpyAsync(&bad_h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  TAMOE_CUDA(cudaStreamSynchronize(s));
  require(bad_h == 0, "non-finite gate logit");

  // topk_route (trainer.cpp:249-250)
  rw.upload_caps(a.caps, s);
  route_rows_from_probs(probs, dm, rw.row_out(nullptr, nullptr), s);
  if (a.aux_kind == 2) {
    // apply_compulsory_quota (trainer.cpp:121-169): quota_i = LRR(c_hat_i / sum(c_hat_i) * S, S); tokens by
    // score claim experts in probability order; every token kept, gate value = the claimed probability
    std::vector<int> q(static_cast<size_t>(P) * N);
    for (int i = 0; i < P; ++i) {
      const double* row = a.c_hat + static_cast<size_t>(i) * N;
      double sum = 0.0;
      for (int e = 0; e < N; ++e) sum += row[e];
      std::vector<double> share(static_cast<size_t>(N));
      for (int e = 0; e < N; ++e) share[static_cast<size_t>(e)] = row[e] / sum * static_cast<double>(S);
      const auto lrr = largest_remainder_round(share.data(), N, S);
      for (int e = 0; e < N; ++e) q[static_cast<size_t>(i) * N + e] = static_cast<int>(lrr[static_cast<size_t>(e)]);
    }
    Scratch<int> quota(static_cast<long long>(P) * N, s);
    const size_t ws_bytes = compulsory_workspace_bytes(P, S);
    Scratch<unsigned char> ws(static_cast<long long>(ws_bytes), s);
    TAMOE_CUDA(cudaMemcpyAsync(quota.p, q.data(), sizeof(int) * q.size(), cudaMemcpyHostToDevice, s));
    route_compulsory(dm, rw.buf, probs, quota.p, ws.p, ws_bytes, s);
    TAMOE_CUDA(cudaMemcpyAsync(rw.buf.gate64, rw.buf.score, sizeof(double) * dm.picks(), cudaMemcpyDeviceToDevice, s));
    rw.finish(0, s);
    TAMOE_CUDA(cudaStreamSynchronize(s));  // q is host memory
  } else {
    rw.finish(a.cap_mode, s);
  }
  const int loss_kind = a.aux_kind == 1 ? 1 : 0;  // compulsory trains with the balance loss (trainer.cpp:253)

  Scratch<double> out(picks * dout, s), resid(T * dout, s), dldg(picks, s), task_part(T, s), dz(T * N, s),
      mean(static_cast<long long>(P) * N, s), coeff(static_cast<long long>(P) * N, s), pen(P * N, s), loss_d(2, s);
  if (loss_kind == 1)
    TAMOE_CUDA(cudaMemcpyAsync(pen.p, a.penalty, sizeof(double) * P * N, cudaMemcpyHostToDevice, s));
  const double mse_scale = 2.0 / (static_cast<double>(P) * S * dout);
  const double task_den = static_cast<double>(P) * S * dout;

  const int row_tiles = static_cast<int>((picks + kT - 1) / kT);  // an expert holds at most P*S kept picks
  const int max_rows = static_cast<int>(std::min<long long>(T, picks));
  if (max_rows > 0) {
    const dim3 gf((dout + kT - 1) / kT, std::min(row_tiles, (max_rows + kT - 1) / kT), N);
    expert_fwd_f64_kernel<<<gf, dim3(kT, kT), 0, s>>>(dm, rw.buf, a.x, a.experts, d, dout, out.p);
    TAMOE_CUDA(cudaGetLastError());
    combine_f64_kernel<<<static_cast<unsigned>(T), 128, sizeof(double) * dout, s>>>(
        dm, rw.buf, out.p, a.y, dout, mse_scale, resid.p, a.y_hat, dldg.p, task_part.p);
    TAMOE_CUDA(cudaGetLastError());
  }
  const dim3 gw((dout + kT - 1) / kT, (d + kT - 1) / kT, N);
  expert_wgrad_f64_kernel<<<gw, dim3(kT, kT), 0, s>>>(dm, rw.buf, a.x, resid.p, d, dout, mse_scale, a.expert_grads);
  TAMOE_CUDA(cudaGetLastError());
  aux_f64_kernel<<<1, 256, 0, s>>>(dm, rw.buf, probs, pen.p, loss_kind, task_part.p, task_den, mean.p, coeff.p,
                                   loss_d.p);
  TAMOE_CUDA(cudaGetLastError());
  if (T > 0) {
    gate_dz_f64_kernel<<<static_cast<unsigned>((T + 127) / 128), 128, 0, s>>>(
        dm, rw.buf, probs, dldg.p, coeff.p, a.aux_weight / static_cast<double>(P), dz.p);
    TAMOE_CUDA(cudaGetLastError());
  }
  TAMOE_CUDA(cudaMemsetAsync(a.gate_grads, 0, sizeof(double) * P * d * N, s));
  for (int i = 0; i < P; ++i)
    add_atb_f64(a.gate_grads + static_cast<long long>(i) * d * N, a.x + static_cast<long long>(i) * S * d,
                dz.p + static_cast<long long>(i) * S * N, S, d, N, s);
  TAMOE_CUDA(cudaMemcpyAsync(a.losses, loss_d.p, sizeof(double) * 2, cudaMemcpyDeviceToHost, s));
  TAMOE_CUDA(cudaStreamSynchronize(s));
  if (!std::isfinite(a.losses[0] + a.aux_weight * a.losses[1]))
    throw std::runtime_error("training diverged (non-finite task / aux loss); lower the learning rate");
}

}  // namespace tamoe
