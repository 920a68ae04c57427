/*
 * TEST INFRASTRUCTURE ONLY -- fp64 restatement of the reference TA-MoE CPU path.
 * See tamoe_oracle.h for the contract.  Each function cites the reference
 * file:line it restates (paths relative to /root/reference/proj/core/src).
 */
#include "tamoe_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

const char* orc_last_error(void) { return g_err; }

static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 2;
}

/* gate.cpp:12-28: max-subtract, exp, sequential sum over e, divide. */
int orc_softmax_rows(const double* logits, int S, int N, double* probs) {
  for (int s = 0; s < S; ++s) {
    const double* l = logits + (size_t)s * N;
    double* p = probs + (size_t)s * N;
    double mx = -INFINITY;
    for (int e = 0; e < N; ++e) {
      if (!isfinite(l[e])) return fail("non-finite gate logit");
      if (l[e] > mx) mx = l[e];
    }
    double denom = 0.0;
    for (int e = 0; e < N; ++e) {
      p[e] = exp(l[e] - mx);
      denom += p[e];
    }
    for (int e = 0; e < N; ++e) p[e] /= denom;
  }
  return 0;
}

/* matrix.hpp:82-93 */
void orc_matmul(const double* a, const double* b, int n, int kdim, int m, double* c) {
  memset(c, 0, sizeof(double) * (size_t)n * m);
  for (int i = 0; i < n; ++i)
    for (int kk = 0; kk < kdim; ++kk) {
      const double aik = a[(size_t)i * kdim + kk];
      if (aik == 0.0) continue;
      for (int j = 0; j < m; ++j) c[(size_t)i * m + j] += aik * b[(size_t)kk * m + j];
    }
}

/* matrix.hpp:96-104: C += alpha A^T B, A [rows x ac], B [rows x bc], C [ac x bc] */
static void add_atb(double* c, const double* a, const double* b, int rows, int ac, int bc, double alpha) {
  for (int kk = 0; kk < rows; ++kk)
    for (int i = 0; i < ac; ++i) {
      const double w = alpha * a[(size_t)kk * ac + i];
      if (w == 0.0) continue;
      for (int j = 0; j < bc; ++j) c[(size_t)i * bc + j] += w * b[(size_t)kk * bc + j];
    }
}

/* gate.cpp:30-32 */
int orc_gate_forward(const double* x, const double* W, int S, int d, int N, double* probs) {
  double* logits = (double*)malloc(sizeof(double) * (size_t)S * N + 1);
  orc_matmul(x, W, S, d, N, logits);
  int rc = orc_softmax_rows(logits, S, N, probs);
  free(logits);
  return rc;
}

/* gate.cpp:52-78 */
typedef struct {
  double rem;
  int idx;
} rem_t;

static int cmp_rem(const void* pa, const void* pb) {
  const rem_t* a = (const rem_t*)pa;
  const rem_t* b = (const rem_t*)pb;
  if (a->rem != b->rem) return a->rem > b->rem ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

void orc_largest_remainder_round(const double* values, int n, long long target, long long* out) {
  rem_t* r = (rem_t*)malloc(sizeof(rem_t) * (size_t)(n + 1));
  long long assigned = 0;
  for (int i = 0; i < n; ++i) {
    const double v = values[i] > 0.0 ? values[i] : 0.0;
    out[i] = (long long)floor(v + 1e-9);
    assigned += out[i];
    r[i].rem = v - (double)out[i];
    r[i].idx = i;
  }
  qsort(r, (size_t)n, sizeof(rem_t), cmp_rem);
  long long left = target - assigned;
  for (int j = 0; j < n && left > 0; ++j, --left) out[r[j].idx] += 1;
  for (int j = n - 1; j >= 0 && left < 0; --j)
    if (out[r[j].idx] > 0) {
      out[r[j].idx] -= 1;
      ++left;
    }
  free(r);
}

typedef struct {
  int process, token, slot;
  double score;
} pick_t;

/* gate.cpp:140-149: score desc, process asc, token asc */
static int cmp_pick(const void* pa, const void* pb) {
  const pick_t* a = (const pick_t*)pa;
  const pick_t* b = (const pick_t*)pb;
  if (a->score != b->score) return a->score > b->score ? -1 : 1;
  if (a->process != b->process) return a->process < b->process ? -1 : 1;
  return a->token < b->token ? -1 : (a->token > b->token);
}

/* gate.cpp:91-202 */
int orc_topk_route(const double* probs, int P, int S, int N, int k, int mode, double cf, const double* c_hat,
                   int* expert, double* gate, double* score, unsigned char* kept, long long* counts,
                   long long* dropped, double* mean_probs) {
  if (P < 1) return fail("topk_route needs at least one process");
  if (k < 1 || k > N) return fail("k must be in [1, N]");
  if (mode == ORC_CAP_PROPORTIONAL && c_hat == NULL)
    return fail("local_proportional capacity requires a target pattern");

  for (int i = 0; i < P; ++i) {
    const double* pr = probs + (size_t)i * S * N;
    double* mp = mean_probs + (size_t)i * N;
    for (int e = 0; e < N; ++e) mp[e] = 0.0;
    for (int s = 0; s < S; ++s) {
      const double* row = pr + (size_t)s * N;
      for (int e = 0; e < N; ++e) mp[e] += row[e] / S;
      /* top-k: higher prob first, ties -> lower expert (gate.cpp:117-122) */
      int sel[64];
      int nsel = 0;
      for (int slot = 0; slot < k; ++slot) {
        int best = -1;
        for (int e = 0; e < N; ++e) {
          int used = 0;
          for (int q = 0; q < nsel; ++q) used |= (sel[q] == e);
          if (used) continue;
          if (best < 0 || row[e] > row[best]) best = e;
        }
        sel[nsel++] = best;
      }
      double mass = 0.0;
      for (int slot = 0; slot < k; ++slot) mass += row[sel[slot]];
      for (int slot = 0; slot < k; ++slot) {
        const size_t a = ((size_t)i * S + s) * k + slot;
        expert[a] = sel[slot];
        score[a] = row[sel[slot]];
        gate[a] = k == 1 ? row[sel[slot]] : row[sel[slot]] / mass;
        kept[a] = 1;
      }
    }
  }

  if (mode != ORC_CAP_NONE) {
    const double cap_real = cf * (double)k * S * P / N; /* gate.hpp:46-48 */
    pick_t* picks = (pick_t*)malloc(sizeof(pick_t) * ((size_t)P * S * k + 1));
    long long* caps = (long long*)malloc(sizeof(long long) * (size_t)(P + 1));
    double* w = (double*)malloc(sizeof(double) * (size_t)(P + 1));
    for (int e = 0; e < N; ++e) {
      int nb = mode == ORC_CAP_GLOBAL ? 1 : P;
      if (mode == ORC_CAP_GLOBAL) {
        caps[0] = (long long)floor(cap_real + 1e-9);
      } else if (mode == ORC_CAP_LOCAL) {
        for (int i = 0; i < P; ++i) caps[i] = (long long)floor(cap_real / P + 1e-9);
      } else {
        double col = 0.0;
        for (int i = 0; i < P; ++i) {
          w[i] = c_hat[(size_t)i * N + e];
          col += c_hat[(size_t)i * N + e];
        }
        if (!(col > 0.0)) {
          free(picks); free(caps); free(w);
          return fail("target pattern column sums to zero");
        }
        for (int i = 0; i < P; ++i) w[i] *= cap_real / col;
        orc_largest_remainder_round(w, P, (long long)floor(cap_real + 1e-9), caps);
      }
      for (int bk = 0; bk < nb; ++bk) {
        size_t np = 0;
        const int i0 = mode == ORC_CAP_GLOBAL ? 0 : bk;
        const int i1 = mode == ORC_CAP_GLOBAL ? P : bk + 1;
        for (int i = i0; i < i1; ++i)
          for (int s = 0; s < S; ++s)
            for (int slot = 0; slot < k; ++slot) {
              const size_t a = ((size_t)i * S + s) * k + slot;
              if (expert[a] == e) {
                picks[np].process = i;
                picks[np].token = s;
                picks[np].slot = slot;
                picks[np].score = score[a];
                ++np;
              }
            }
        qsort(picks, np, sizeof(pick_t), cmp_pick);
        const long long cap = caps[bk] > 0 ? caps[bk] : 0;
        for (size_t q = (size_t)cap; q < np; ++q)
          kept[((size_t)picks[q].process * S + picks[q].token) * k + picks[q].slot] = 0;
      }
    }
    free(picks); free(caps); free(w);
  }

  for (int i = 0; i < P; ++i) {
    for (int e = 0; e < N; ++e) counts[(size_t)i * N + e] = dropped[(size_t)i * N + e] = 0;
    for (int s = 0; s < S; ++s)
      for (int slot = 0; slot < k; ++slot) {
        const size_t a = ((size_t)i * S + s) * k + slot;
        if (kept[a]) counts[(size_t)i * N + expert[a]] += 1;
        else dropped[(size_t)i * N + expert[a]] += 1;
      }
  }
  return 0;
}

/* gate.cpp:209-214 */
double orc_loss_balance(const long long* counts, const double* mean_probs, int N, int S) {
  double loss = 0.0;
  for (int e = 0; e < N; ++e) loss += mean_probs[e] * ((double)counts[e] / S);
  return loss;
}

/* gate.cpp:222-246 */
int orc_penalty_weights(const double* c_hat_row, int n, int norm, double temperature, double* p) {
  double* inv = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  for (int e = 0; e < n; ++e) {
    if (!(c_hat_row[e] > 0.0)) {
      free(inv);
      return fail("penalty weights need strictly positive targets");
    }
    inv[e] = 1.0 / c_hat_row[e];
  }
  if (norm == 0) {
    double total = 0.0;
    for (int e = 0; e < n; ++e) total += inv[e];
    for (int e = 0; e < n; ++e) p[e] = inv[e] / total;
  } else {
    double t = temperature;
    if (!(t > 0.0)) {
      double s = 0.0;
      for (int e = 0; e < n; ++e) s += inv[e];
      t = s / (double)n;
    }
    double zmax = -INFINITY;
    for (int e = 0; e < n; ++e)
      if (inv[e] / t > zmax) zmax = inv[e] / t;
    double denom = 0.0;
    for (int e = 0; e < n; ++e) {
      p[e] = exp(inv[e] / t - zmax);
      denom += p[e];
    }
    for (int e = 0; e < n; ++e) p[e] /= denom;
  }
  free(inv);
  return 0;
}

/* gate.cpp:248-255 */
double orc_loss_topo(const long long* counts, const double* mean_probs, const double* penalty, int N, int P, int S) {
  double loss = 0.0;
  for (int e = 0; e < N; ++e) loss += penalty[e] * mean_probs[e] * ((double)counts[e] / S);
  return (double)N * P * loss;
}

/* gate.cpp:273-278 */
void orc_balance_coefficients(const long long* counts, int N, int S, double* coeff) {
  const double s2 = (double)S * S;
  for (int e = 0; e < N; ++e) coeff[e] = (double)counts[e] / s2;
}

/* gate.cpp:280-287 */
void orc_topo_coefficients(const long long* counts, const double* penalty, int N, int P, int S, double* coeff) {
  const double scale = (double)N * P / ((double)S * S);
  for (int e = 0; e < N; ++e) coeff[e] = scale * penalty[e] * (double)counts[e];
}

/* gate.cpp:257-271 */
void orc_grad_aux_loss(const double* x, const double* probs, const double* coeff, int S, int d, int N, double* grad) {
  double* dz = (double*)malloc(sizeof(double) * (size_t)S * N + 1);
  for (int s = 0; s < S; ++s) {
    const double* p = probs + (size_t)s * N;
    double dot = 0.0;
    for (int e = 0; e < N; ++e) dot += coeff[e] * p[e];
    for (int e = 0; e < N; ++e) dz[(size_t)s * N + e] = p[e] * (coeff[e] - dot);
  }
  memset(grad, 0, sizeof(double) * (size_t)d * N);
  add_atb(grad, x, dz, S, d, N, 1.0);
  free(dz);
}

/* solver.cpp:28-52 (Eq. 8) */
int orc_target_closed_form(const double* beta, int P, int N, int k, int S, double* c_hat) {
  if (k < 1 || S < 1 || N < 1 || P < 1) return fail("k, S, N, P must be positive");
  if (N % P != 0) return fail("N must be divisible by P");
  if (k > N) return fail("k cannot exceed N");
  for (int i = 0; i < P * P; ++i)
    if (!(beta[i] > 0.0)) return fail("closed form requires strictly positive beta_hat");
  const int E = N / P;
  const double row_target = (double)k * S;
  for (int i = 0; i < P; ++i) {
    double inv_sum = 0.0;
    for (int j = 0; j < P; ++j) inv_sum += 1.0 / beta[i * P + j];
    for (int e = 0; e < N; ++e) c_hat[(size_t)i * N + e] = row_target / (E * inv_sum * beta[i * P + e / E]);
  }
  return 0;
}

/* trainer.cpp:121-169 */
typedef struct {
  double key;
  int idx;
} key_t_;

static int cmp_key_desc(const void* pa, const void* pb) {
  const key_t_* a = (const key_t_*)pa;
  const key_t_* b = (const key_t_*)pb;
  if (a->key != b->key) return a->key > b->key ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

int orc_apply_compulsory_quota(const double* probs, const double* c_hat_row, int S, int N, int* expert,
                               double* gate, double* score, unsigned char* kept, long long* counts,
                               long long* dropped) {
  double* share = (double*)calloc((size_t)N + 1, sizeof(double));
  long long* quota = (long long*)malloc(sizeof(long long) * (size_t)N);
  key_t_* order = (key_t_*)malloc(sizeof(key_t_) * (size_t)(S + 1));
  key_t_* er = (key_t_*)malloc(sizeof(key_t_) * (size_t)N);
  double row_sum = 0.0;
  for (int e = 0; e < N; ++e) row_sum += c_hat_row[e];
  for (int e = 0; e < N; ++e) share[e] = c_hat_row[e] / row_sum * (double)S;
  orc_largest_remainder_round(share, N, S, quota);
  for (int s = 0; s < S; ++s) {
    order[s].key = score[s];
    order[s].idx = s;
  }
  qsort(order, (size_t)S, sizeof(key_t_), cmp_key_desc);
  for (int q = 0; q < S; ++q) {
    const int s = order[q].idx;
    const double* p = probs + (size_t)s * N;
    for (int e = 0; e < N; ++e) {
      er[e].key = p[e];
      er[e].idx = e;
    }
    qsort(er, (size_t)N, sizeof(key_t_), cmp_key_desc);
    for (int r = 0; r < N; ++r) {
      const int e = er[r].idx;
      if (quota[e] > 0) {
        quota[e] -= 1;
        expert[s] = e;
        score[s] = p[e];
        gate[s] = p[e];
        kept[s] = 1;
        break;
      }
    }
  }
  for (int e = 0; e < N; ++e) counts[e] = dropped[e] = 0;
  for (int s = 0; s < S; ++s) counts[expert[s]] += 1;
  free(share); free(quota); free(order); free(er);
  return 0;
}

/* ------------------------------------------------------------------ layer step */
static double act_f(int act, double x) {
  if (act == ORC_ACT_GELU) {
    const double k0 = 0.7978845608028654, k1 = 0.044715;
    return 0.5 * x * (1.0 + tanh(k0 * (x + k1 * x * x * x)));
  }
  if (act == ORC_ACT_RELU) return x > 0.0 ? x : 0.0;
  return x;
}
static double act_g(int act, double x) {
  if (act == ORC_ACT_GELU) {
    const double k0 = 0.7978845608028654, k1 = 0.044715;
    const double t = tanh(k0 * (x + k1 * x * x * x));
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * k0 * (1.0 + 3.0 * k1 * x * x);
  }
  if (act == ORC_ACT_RELU) return x > 0.0 ? 1.0 : 0.0;
  return 1.0;
}

/* trainer.cpp:371-482 (one step, all processes; no SGD update) */
int orc_layer_step(const orc_layer_cfg* c, const double* x, const double* y, const double* gates, const double* U,
                   const double* W1, const double* W2, orc_layer_out* o) {
  const int P = c->P, S = c->S, d = c->d, dout = c->d_out, N = c->N, k = c->k, f = c->f;
  if (k < 1 || k > N || k > 64) return fail("k must be in [1, N]");
  if (c->aux_kind == ORC_AUX_TOPO && c->penalties == NULL) return fail("topo loss requires penalties");
  const size_t PSk = (size_t)P * S * k;
  double* probs = o->probs ? o->probs : (double*)malloc(sizeof(double) * (size_t)P * S * N);
  int* expert = o->expert ? o->expert : (int*)malloc(sizeof(int) * PSk);
  double* gate = o->gate ? o->gate : (double*)malloc(sizeof(double) * PSk);
  double* score = o->score ? o->score : (double*)malloc(sizeof(double) * PSk);
  unsigned char* kept = o->kept ? o->kept : (unsigned char*)malloc(PSk);
  long long* counts = o->counts ? o->counts : (long long*)malloc(sizeof(long long) * (size_t)P * N);
  long long* dropped = o->dropped ? o->dropped : (long long*)malloc(sizeof(long long) * (size_t)P * N);
  double* mean_probs = o->mean_probs ? o->mean_probs : (double*)malloc(sizeof(double) * (size_t)P * N);
  int rc = 0;

  for (int i = 0; i < P && rc == 0; ++i)
    rc = orc_gate_forward(x + (size_t)i * S * d, gates + (size_t)i * d * N, S, d, N, probs + (size_t)i * S * N);
  if (rc == 0)
    rc = orc_topk_route(probs, P, S, N, k, c->cap_mode, c->cf, c->c_hat, expert, gate, score, kept, counts, dropped,
                        mean_probs);
  if (rc != 0) goto done;

  {
    const double mse_scale = 2.0 / ((double)P * S * dout); /* trainer.cpp:243 */
    double step_task = 0.0, step_aux = 0.0;
    double* dpi = (double*)malloc(sizeof(double) * (size_t)S * N);
    double* dz = (double*)malloc(sizeof(double) * (size_t)S * N);
    double* resid = (double*)malloc(sizeof(double) * (size_t)dout);
    double* outs = (double*)malloc(sizeof(double) * (size_t)k * dout);
    double* hid = f > 0 ? (double*)malloc(sizeof(double) * (size_t)k * f) : NULL;
    double* pre = f > 0 ? (double*)malloc(sizeof(double) * (size_t)k * f) : NULL;
    double* go = (double*)malloc(sizeof(double) * (size_t)dout);
    double* dh = f > 0 ? (double*)malloc(sizeof(double) * (size_t)f) : NULL;
    double* dldg = (double*)malloc(sizeof(double) * (size_t)k);
    double* coeff = (double*)malloc(sizeof(double) * (size_t)N);
    if (o->grad_u) memset(o->grad_u, 0, sizeof(double) * (size_t)N * d * dout);
    if (o->grad_w1) memset(o->grad_w1, 0, sizeof(double) * (size_t)N * d * (size_t)(f > 0 ? f : 0));
    if (o->grad_w2) memset(o->grad_w2, 0, sizeof(double) * (size_t)N * (size_t)(f > 0 ? f : 0) * dout);
    if (o->dx) memset(o->dx, 0, sizeof(double) * (size_t)P * S * d);

    for (int i = 0; i < P; ++i) {
      const double* xi = x + (size_t)i * S * d;
      const double* yi = y + (size_t)i * S * dout;
      const double* pi = probs + (size_t)i * S * N;
      memset(dpi, 0, sizeof(double) * (size_t)S * N);
      for (int s = 0; s < S; ++s) {
        const double* xs = xi + (size_t)s * d;
        const size_t a0 = ((size_t)i * S + s) * k;
        for (int j = 0; j < dout; ++j) resid[j] = 0.0;
        for (int slot = 0; slot < k; ++slot) {
          if (!kept[a0 + slot]) continue;
          const int e = expert[a0 + slot];
          double* ov = outs + (size_t)slot * dout;
          for (int j = 0; j < dout; ++j) ov[j] = 0.0;
          if (f == 0) { /* trainer.cpp:284-289 */
            const double* u = U + (size_t)e * d * dout;
            for (int r = 0; r < d; ++r) {
              const double xr = xs[r];
              if (xr == 0.0) continue;
              for (int j = 0; j < dout; ++j) ov[j] += xr * u[(size_t)r * dout + j];
            }
          } else {
            const double* w1 = W1 + (size_t)e * d * f;
            const double* w2 = W2 + (size_t)e * f * dout;
            double* a = pre + (size_t)slot * f;
            double* h = hid + (size_t)slot * f;
            for (int q = 0; q < f; ++q) a[q] = 0.0;
            for (int r = 0; r < d; ++r) {
              const double xr = xs[r];
              if (xr == 0.0) continue;
              for (int q = 0; q < f; ++q) a[q] += xr * w1[(size_t)r * f + q];
            }
            for (int q = 0; q < f; ++q) h[q] = act_f(c->act, a[q]);
            for (int q = 0; q < f; ++q) {
              const double hq = h[q];
              if (hq == 0.0) continue;
              for (int j = 0; j < dout; ++j) ov[j] += hq * w2[(size_t)q * dout + j];
            }
          }
          for (int j = 0; j < dout; ++j) resid[j] += gate[a0 + slot] * ov[j]; /* trainer.cpp:290-291 */
        }
        if (o->y_hat)
          for (int j = 0; j < dout; ++j) o->y_hat[((size_t)i * S + s) * dout + j] = resid[j];
        for (int j = 0; j < dout; ++j) {
          resid[j] -= yi[(size_t)s * dout + j];
          step_task += resid[j] * resid[j];
        }
        /* trainer.cpp:298-316 */
        double mass = 0.0;
        for (int slot = 0; slot < k; ++slot) mass += score[a0 + slot];
        for (int slot = 0; slot < k; ++slot) {
          dldg[slot] = 0.0;
          if (!kept[a0 + slot]) continue;
          const int e = expert[a0 + slot];
          const double* ov = outs + (size_t)slot * dout;
          double dot = 0.0;
          for (int j = 0; j < dout; ++j) dot += resid[j] * ov[j];
          dldg[slot] = mse_scale * dot;
          const double g = gate[a0 + slot];
          if (f == 0) {
            if (o->grad_u) {
              double* ug = o->grad_u + (size_t)e * d * dout;
              for (int r = 0; r < d; ++r) {
                const double xr = mse_scale * g * xs[r];
                if (xr == 0.0) continue;
                for (int j = 0; j < dout; ++j) ug[(size_t)r * dout + j] += xr * resid[j];
              }
            }
            if (o->dx) { /* extension: dx += U (mse_scale g r) */
              const double* u = U + (size_t)e * d * dout;
              for (int r = 0; r < d; ++r) {
                double acc = 0.0;
                for (int j = 0; j < dout; ++j) acc += u[(size_t)r * dout + j] * (mse_scale * g * resid[j]);
                o->dx[((size_t)i * S + s) * d + r] += acc;
              }
            }
          } else { /* extension: two-layer FFN backward */
            const double* w1 = W1 + (size_t)e * d * f;
            const double* w2 = W2 + (size_t)e * f * dout;
            const double* a = pre + (size_t)slot * f;
            const double* h = hid + (size_t)slot * f;
            for (int j = 0; j < dout; ++j) go[j] = mse_scale * g * resid[j];
            if (o->grad_w2) {
              double* g2 = o->grad_w2 + (size_t)e * f * dout;
              for (int q = 0; q < f; ++q)
                for (int j = 0; j < dout; ++j) g2[(size_t)q * dout + j] += h[q] * go[j];
            }
            for (int q = 0; q < f; ++q) {
              double acc = 0.0;
              for (int j = 0; j < dout; ++j) acc += w2[(size_t)q * dout + j] * go[j];
              dh[q] = acc * act_g(c->act, a[q]);
            }
            if (o->grad_w1) {
              double* g1 = o->grad_w1 + (size_t)e * d * f;
              for (int r = 0; r < d; ++r)
                for (int q = 0; q < f; ++q) g1[(size_t)r * f + q] += xs[r] * dh[q];
            }
            if (o->dx)
              for (int r = 0; r < d; ++r) {
                double acc = 0.0;
                for (int q = 0; q < f; ++q) acc += w1[(size_t)r * f + q] * dh[q];
                o->dx[((size_t)i * S + s) * d + r] += acc;
              }
          }
        }
        /* trainer.cpp:318-331 */
        if (k == 1) {
          if (kept[a0]) dpi[(size_t)s * N + expert[a0]] += dldg[0];
        } else {
          for (int l = 0; l < k; ++l) {
            double acc = 0.0;
            for (int j = 0; j < k; ++j) {
              if (dldg[j] == 0.0) continue;
              const double del = j == l ? mass : 0.0;
              acc += dldg[j] * (del - score[a0 + j]) / (mass * mass);
            }
            dpi[(size_t)s * N + expert[a0 + l]] += acc;
          }
        }
      }
      /* trainer.cpp:334-345 */
      const long long* ci = counts + (size_t)i * N;
      const double* mi = mean_probs + (size_t)i * N;
      if (c->aux_kind == ORC_AUX_TOPO) {
        const double* pen = c->penalties + (size_t)i * N;
        step_aux += orc_loss_topo(ci, mi, pen, N, P, S);
        orc_topo_coefficients(ci, pen, N, P, S, coeff);
      } else {
        step_aux += orc_loss_balance(ci, mi, N, S);
        orc_balance_coefficients(ci, N, S, coeff);
      }
      const double aux_scale = c->aux_weight / (double)P;
      for (int s = 0; s < S; ++s)
        for (int e = 0; e < N; ++e) dpi[(size_t)s * N + e] += aux_scale * coeff[e];
      /* trainer.cpp:347-355 */
      for (int s = 0; s < S; ++s) {
        double dot = 0.0;
        for (int e = 0; e < N; ++e) dot += dpi[(size_t)s * N + e] * pi[(size_t)s * N + e];
        for (int e = 0; e < N; ++e)
          dz[(size_t)s * N + e] = pi[(size_t)s * N + e] * (dpi[(size_t)s * N + e] - dot);
      }
      if (o->gate_grads) {
        double* gg = o->gate_grads + (size_t)i * d * N;
        memset(gg, 0, sizeof(double) * (size_t)d * N);
        add_atb(gg, xi, dz, S, d, N, 1.0);
      }
      if (o->dx) { /* extension: dx += dz W^T */
        const double* Wi = gates + (size_t)i * d * N;
        for (int s = 0; s < S; ++s)
          for (int r = 0; r < d; ++r) {
            double acc = 0.0;
            for (int e = 0; e < N; ++e) acc += dz[(size_t)s * N + e] * Wi[(size_t)r * N + e];
            o->dx[((size_t)i * S + s) * d + r] += acc;
          }
      }
    }
    o->task_loss = step_task / ((double)P * S * dout);
    o->aux_loss = step_aux / (double)P;
    free(dpi); free(dz); free(resid); free(outs); free(hid); free(pre); free(go); free(dh); free(dldg); free(coeff);
  }

done:
  if (!o->probs) free(probs);
  if (!o->expert) free(expert);
  if (!o->gate) free(gate);
  if (!o->score) free(score);
  if (!o->kept) free(kept);
  if (!o->counts) free(counts);
  if (!o->dropped) free(dropped);
  if (!o->mean_probs) free(mean_probs);
  return rc;
}
