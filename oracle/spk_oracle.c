/*
 * spk_oracle.c -- CPU restatement of the reference's Spar-Sink hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see spk_oracle.h). Plain C99, single thread,
 * sequential sums in the reference's order, built with -O2
 * -ffp-contract=off so no FMA is formed (the reference's -O2 x86-64 build
 * has none either). Citations are /root/reference/proj file:line.
 */
#define _POSIX_C_SOURCE 200809L
#include "spk_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define KPI 3.14159265358979323846
#define GOLDEN 0x9e3779b97f4a7c15ULL

static void set_msg(char* msg, size_t len, const char* cls, const char* text) {
  if (msg && len) snprintf(msg, len, "%s%s%s", cls ? cls : "", cls ? ": " : "", text);
}

/* ---- RNG ------------------------------------------------------------------ */

/* rng.hpp:10-15 */
uint64_t spko_splitmix64(uint64_t x) {
  x += GOLDEN;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* rng.hpp:17-19 */
uint64_t spko_mix_seed(uint64_t seed, uint64_t stream) {
  return spko_splitmix64(seed ^ spko_splitmix64(stream + 0x632be59bd9b4e019ULL));
}

/* CounterRng: state starts at mix_seed(seed, stream) (rng.hpp:26-27); the
 * t-th next_u64 adds t*GOLDEN and applies the splitmix finalizer without its
 * own increment (rng.hpp:29-35); next_double keeps the top 53 bits
 * (rng.hpp:38-40). Closed form of the t-th draw. */
double spko_counter_draw(uint64_t seed, uint64_t stream, uint64_t t) {
  uint64_t x = spko_mix_seed(seed, stream) + t * GOLDEN;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  x = x ^ (x >> 31);
  return (double)(x >> 11) * 0x1.0p-53;
}

void spko_rng_doubles(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  for (int64_t k = 0; k < count; ++k) out[k] = spko_counter_draw(seed, stream, (uint64_t)k + 1);
}

/* rng.cpp:7-21 (Box-Muller, cos first, sin kept as the spare) */
void spko_rng_normals(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  uint64_t t = 0;
  for (int64_t k = 0; k < count; k += 2) {
    double u1 = spko_counter_draw(seed, stream, ++t);
    double u2 = spko_counter_draw(seed, stream, ++t);
    if (u1 < 1e-300) u1 = 1e-300;
    const double r = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    out[k] = r * cos(theta);
    if (k + 1 < count) out[k + 1] = r * sin(theta);
  }
}

/* ---- measures.cpp:12-34 ------------------------------------------------- */

int spko_new_measure(const double* w, int64_t n, int require_simplex, double* total) {
  if (n <= 0) return SPKO_E_LENGTH_MISMATCH;
  double tot = 0.0;
  int any_positive = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (w[i] < 0.0 || !isfinite(w[i])) return SPKO_E_NEGATIVE_WEIGHT;
    any_positive = any_positive || w[i] > 0.0;
    tot += w[i];
  }
  if (!any_positive) return SPKO_E_NEGATIVE_WEIGHT;
  if (require_simplex && fabs(tot - 1.0) > 1e-8) return SPKO_E_NOT_NORMALIZED;
  *total = tot;
  return SPKO_OK;
}

/* ---- geometry.cpp ----------------------------------------------------------- */

/* sq_dist geometry.cpp:16-23 + the per-kind switch :41-59 */
double spko_cost_entry(const double* p, const double* q, int dim, int kind, double eta) {
  double d2 = 0.0;
  for (int k = 0; k < dim; ++k) {
    const double diff = p[k] - q[k];
    d2 += diff * diff;
  }
  if (kind == SPKO_COST_SQEUCLID) return d2;
  if (kind == SPKO_COST_EUCLID) return sqrt(d2);
  {
    const double d = sqrt(d2);
    if (d >= KPI * eta) return INFINITY;
    const double cz = cos(d / (2.0 * eta));
    double v = -log(cz * cz);
    if (!(v >= 0.0)) v = 0.0;
    return v;
  }
}

/* geometry.cpp:25-66 (+ wfr_cost's eta check :78-81) */
int spko_pairwise_cost(const double* x, int64_t nx, const double* y, int64_t ny, int dim,
                       int kind, double eta, double* C, double* c0_out) {
  if (dim <= 0) return SPKO_E_DIMENSION_MISMATCH;
  if (kind == SPKO_COST_WFR && !(eta > 0.0)) return SPKO_E_NON_POSITIVE_ETA;
  double c0 = 0.0;
  for (int64_t i = 0; i < nx; ++i) {
    for (int64_t j = 0; j < ny; ++j) {
      const double v = spko_cost_entry(x + i * dim, y + j * dim, dim, kind, eta);
      C[i * ny + j] = v;
      if (isfinite(v) && v > c0) c0 = v;
    }
  }
  if (c0_out) *c0_out = c0;
  return SPKO_OK;
}

/* geometry.cpp:83-102 */
int spko_kernel_from_cost(const double* C, int64_t rows, int64_t cols, double eps, double* K,
                          double* nnz_ratio) {
  if (!(eps > 0.0)) return SPKO_E_NON_POSITIVE_EPSILON;
  int64_t nnz = 0;
  for (int64_t i = 0; i < rows * cols; ++i) {
    const double v = isinf(C[i]) ? 0.0 : exp(-C[i] / eps);
    K[i] = v;
    nnz += v > 0.0 ? 1 : 0;
  }
  *nnz_ratio = (double)nnz / (double)(rows * cols);
  return SPKO_OK;
}

/* ---- plans -------------------------------------------------------------------- */

void spko_plan_free(spko_plan* p) {
  if (!p) return;
  free(p->grid);
  free(p->row_w);
  free(p->col_w);
  p->grid = p->row_w = p->col_w = NULL;
}

/* sparsify.hpp:28-34 */
double spko_plan_prob(const spko_plan* p, int64_t i, int64_t j) {
  const double base = p->grid ? p->grid[i * p->n + j] : p->row_w[i] * p->col_w[j];
  if (p->theta == 0.0) return base;
  return base == 0.0 ? 0.0 : (1.0 - p->theta) * base + p->theta / (double)p->kernel_nnz;
}

/* sparsify.cpp:36-39 */
static int64_t kernel_nnz_count(int64_t n, double nnz_ratio) {
  return (int64_t)llround(nnz_ratio * (double)n * (double)n);
}

/* sparsify.cpp:49-67: zero the grid off the support, sequential row-major
 * total, multiply by the reciprocal. */
static int masked_grid_plan(int kind, int64_t n, double* grid, const double* K,
                            spko_plan* out) {
  double total = 0.0;
  int64_t nnz = 0;
  for (int64_t i = 0; i < n; ++i) {
    double* prow = grid + i * n;
    const double* krow = K + i * n;
    for (int64_t j = 0; j < n; ++j) {
      if (krow[j] == 0.0) prow[j] = 0.0;
      total += prow[j];
      nnz += krow[j] > 0.0 ? 1 : 0;
    }
  }
  if (total <= 0.0) {
    free(grid);
    return SPKO_E_ALL_ZERO_KERNEL;
  }
  const double inv = 1.0 / total;
  for (int64_t k = 0; k < n * n; ++k) grid[k] *= inv;
  memset(out, 0, sizeof *out);
  out->kind = kind;
  out->n = n;
  out->factorized = 0;
  out->kernel_nnz = nnz;
  out->grid = grid;
  return SPKO_OK;
}

/* sparsify.cpp:71-91 (check_sizes :41-46 folded in by the caller sizes) */
int spko_ot_probabilities(const double* a, const double* b, int64_t n, const double* K,
                          double nnz_ratio, spko_plan* out) {
  if (kernel_nnz_count(n, nnz_ratio) == 0) return SPKO_E_ALL_ZERO_KERNEL;
  double* ra = (double*)malloc(sizeof(double) * n);
  double* cb = (double*)malloc(sizeof(double) * n);
  double sa = 0.0, sb = 0.0;
  for (int64_t i = 0; i < n; ++i) sa += (ra[i] = sqrt(a[i]));
  for (int64_t j = 0; j < n; ++j) sb += (cb[j] = sqrt(b[j]));
  if (sa == 0.0 || sb == 0.0) {
    free(ra);
    free(cb);
    return SPKO_E_ALL_ZERO_KERNEL;
  }
  for (int64_t i = 0; i < n; ++i) ra[i] /= sa;
  for (int64_t j = 0; j < n; ++j) cb[j] /= sb;
  if (nnz_ratio == 1.0) {
    memset(out, 0, sizeof *out);
    out->kind = SPKO_PLAN_OT;
    out->n = n;
    out->factorized = 1;
    out->kernel_nnz = n * n;
    out->row_w = ra;
    out->col_w = cb;
    return SPKO_OK;
  }
  double* grid = (double*)malloc(sizeof(double) * n * n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) grid[i * n + j] = ra[i] * cb[j];
  free(ra);
  free(cb);
  return masked_grid_plan(SPKO_PLAN_OT, n, grid, K, out);
}

/* sparsify.cpp:93-115 */
int spko_uot_probabilities(const double* a, const double* b, int64_t n, const double* K,
                           double nnz_ratio, double lambda, double eps, spko_plan* out) {
  if (!(lambda > 0.0)) return SPKO_E_ERROR;
  if (!(eps > 0.0)) return SPKO_E_NON_POSITIVE_EPSILON;
  if (kernel_nnz_count(n, nnz_ratio) == 0) return SPKO_E_ALL_ZERO_KERNEL;
  const double g_ab = lambda / (2.0 * lambda + eps);
  const double g_k = eps / (2.0 * lambda + eps);
  double* pa = (double*)malloc(sizeof(double) * n);
  double* pb = (double*)malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) pa[i] = pow(a[i], g_ab);
  for (int64_t j = 0; j < n; ++j) pb[j] = pow(b[j], g_ab);
  double* grid = (double*)malloc(sizeof(double) * n * n);
  for (int64_t i = 0; i < n; ++i) {
    const double* krow = K + i * n;
    double* prow = grid + i * n;
    for (int64_t j = 0; j < n; ++j)
      prow[j] = krow[j] > 0.0 ? pa[i] * pb[j] * pow(krow[j], g_k) : 0.0;
  }
  free(pa);
  free(pb);
  return masked_grid_plan(SPKO_PLAN_UOT, n, grid, K, out);
}

/* sparsify.cpp:137-147 */
int spko_uniform_probabilities(int64_t n, const double* K, double nnz_ratio, spko_plan* out) {
  if (kernel_nnz_count(n, nnz_ratio) == 0) return SPKO_E_ALL_ZERO_KERNEL;
  if (nnz_ratio == 1.0) {
    double* rw = (double*)malloc(sizeof(double) * n);
    double* cw = (double*)malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) rw[i] = cw[i] = 1.0 / (double)n;
    memset(out, 0, sizeof *out);
    out->kind = SPKO_PLAN_UNIFORM;
    out->n = n;
    out->factorized = 1;
    out->kernel_nnz = n * n;
    out->row_w = rw;
    out->col_w = cw;
    return SPKO_OK;
  }
  double* grid = (double*)malloc(sizeof(double) * n * n);
  for (int64_t k = 0; k < n * n; ++k) grid[k] = 1.0;
  return masked_grid_plan(SPKO_PLAN_UNIFORM, n, grid, K, out);
}

/* sparsify.cpp:149-167 */
int spko_shrink_with_uniform(spko_plan* p, double theta) {
  if (!(theta >= 0.0 && theta < 1.0)) return SPKO_E_THETA_OUT_OF_RANGE;
  if (theta == 0.0) {
    p->theta = 0.0;
    return SPKO_OK;
  }
  if (p->grid) {
    const double unif = theta / (double)p->kernel_nnz;
    for (int64_t k = 0; k < p->n * p->n; ++k)
      if (p->grid[k] > 0.0) p->grid[k] = (1.0 - theta) * p->grid[k] + unif;
    p->theta = 0.0;
  } else {
    p->theta = theta;
  }
  return SPKO_OK;
}

/* ---- sketch ------------------------------------------------------------------ */

void spko_csr_free(spko_csr* s) {
  if (!s) return;
  free(s->row_ptr);
  free(s->col_idx);
  free(s->values);
  s->row_ptr = NULL;
  s->col_idx = NULL;
  s->values = NULL;
}

typedef struct {
  int64_t cap, nnz;
  uint32_t* col;
  double* val;
} growbuf;

static void gb_push(growbuf* g, uint32_t c, double v) {
  if (g->nnz == g->cap) {
    g->cap = g->cap ? g->cap * 2 : 1024;
    g->col = (uint32_t*)realloc(g->col, sizeof(uint32_t) * g->cap);
    g->val = (double*)realloc(g->val, sizeof(double) * g->cap);
  }
  g->col[g->nnz] = c;
  g->val[g->nnz] = v;
  g->nnz++;
}

/* sparsify.cpp:169-201. Row i uses CounterRng(seed, i); one draw per entry
 * with K_ij != 0 (drawn even when p* <= 0); keep when draw < p*; store
 * p* >= 1 ? K : K/p*. */
int spko_poisson_sparsify(const double* K, int64_t n, const spko_plan* plan, double s,
                          uint64_t seed, spko_csr* out) {
  if (plan->n != n) return SPKO_E_LENGTH_MISMATCH;
  if (!(s > 0.0) || s >= (double)n * (double)n) return SPKO_E_BUDGET_TOO_LARGE;
  growbuf g = {0, 0, NULL, NULL};
  int64_t* rp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t state0 = spko_mix_seed(seed, (uint64_t)i);
    uint64_t t = 0;
    const double* krow = K + i * n;
    for (int64_t j = 0; j < n; ++j) {
      if (krow[j] == 0.0) continue;
      const double sp = s * spko_plan_prob(plan, i, j);
      const double p_star = (sp < 1.0) ? sp : 1.0; /* std::min(1.0, sp) */
      ++t;
      uint64_t x = state0 + t * GOLDEN;
      x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
      x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
      x = x ^ (x >> 31);
      const double draw = (double)(x >> 11) * 0x1.0p-53;
      if (p_star <= 0.0) continue;
      if (draw < p_star) gb_push(&g, (uint32_t)j, p_star >= 1.0 ? krow[j] : krow[j] / p_star);
    }
    rp[i + 1] = g.nnz;
  }
  out->n = n;
  out->nnz = g.nnz;
  out->row_ptr = rp;
  out->col_idx = g.col ? g.col : (uint32_t*)malloc(4);
  out->values = g.val ? g.val : (double*)malloc(8);
  return SPKO_OK;
}

/* sparsify.cpp:203-213 */
void spko_spmv(const spko_csr* M, const double* v, double* out) {
  for (int64_t i = 0; i < M->n; ++i) {
    double acc = 0.0;
    for (int64_t p = M->row_ptr[i]; p < M->row_ptr[i + 1]; ++p)
      acc += M->values[p] * v[M->col_idx[p]];
    out[i] = acc;
  }
}

/* sparsify.cpp:215-226 */
void spko_spmv_t(const spko_csr* M, const double* u, double* out) {
  for (int64_t j = 0; j < M->n; ++j) out[j] = 0.0;
  for (int64_t i = 0; i < M->n; ++i) {
    const double ui = u[i];
    if (ui == 0.0) continue;
    for (int64_t p = M->row_ptr[i]; p < M->row_ptr[i + 1]; ++p)
      out[M->col_idx[p]] += M->values[p] * ui;
  }
}

/* Coordinate restatement of the same draw rule for rows [r0, r1). */
int spko_sample_rows_coords(const double* x, const double* y, int64_t n, int dim,
                            int cost_kind, double eta, double scale, double eps,
                            int plan_kind, int factorized, const double* row_w,
                            const double* col_w, double g_k, double inv, double s,
                            uint64_t seed, int64_t r0, int64_t r1, spko_csr* out) {
  if (!(s > 0.0) || s >= (double)n * (double)n) return SPKO_E_BUDGET_TOO_LARGE;
  growbuf g = {0, 0, NULL, NULL};
  const int64_t rows = r1 - r0;
  int64_t* rp = (int64_t*)calloc((size_t)rows + 1, sizeof(int64_t));
  for (int64_t i = r0; i < r1; ++i) {
    const uint64_t state0 = spko_mix_seed(seed, (uint64_t)i);
    uint64_t t = 0;
    for (int64_t j = 0; j < n; ++j) {
      const double c = spko_cost_entry(x + i * dim, y + j * dim, dim, cost_kind, eta) / scale;
      const double k = isinf(c) ? 0.0 : exp(-c / eps);
      if (k == 0.0) continue;
      double prob;
      if (plan_kind == SPKO_PLAN_UOT) {
        prob = row_w[i] * col_w[j] * pow(k, g_k) * inv;
      } else if (plan_kind == SPKO_PLAN_UNIFORM && !factorized) {
        prob = 1.0 * inv;
      } else {
        prob = factorized ? row_w[i] * col_w[j] : row_w[i] * col_w[j] * inv;
      }
      const double sp = s * prob;
      const double p_star = (sp < 1.0) ? sp : 1.0;
      ++t;
      uint64_t h = state0 + t * GOLDEN;
      h = (h ^ (h >> 30)) * 0xbf58476d1ce4e5b9ULL;
      h = (h ^ (h >> 27)) * 0x94d049bb133111ebULL;
      h = h ^ (h >> 31);
      const double draw = (double)(h >> 11) * 0x1.0p-53;
      if (p_star <= 0.0) continue;
      if (draw < p_star) gb_push(&g, (uint32_t)j, p_star >= 1.0 ? k : k / p_star);
    }
    rp[i - r0 + 1] = g.nnz;
  }
  out->n = rows;
  out->nnz = g.nnz;
  out->row_ptr = rp;
  out->col_idx = g.col ? g.col : (uint32_t*)malloc(4);
  out->values = g.val ? g.val : (double*)malloc(8);
  return SPKO_OK;
}

/* ---- solvers ------------------------------------------------------------------ */

typedef struct {
  const spko_csr* sk;
  const double* K;
  int64_t n;
} kop;

/* kernel_apply (solvers.cpp:12-22 dense, :36-39 sparse) */
static void op_apply(const kop* op, const double* v, double* out) {
  if (op->sk) {
    spko_spmv(op->sk, v, out);
    return;
  }
  const int64_t n = op->n;
  for (int64_t i = 0; i < n; ++i) {
    const double* row = op->K + i * n;
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) acc += row[j] * v[j];
    out[i] = acc;
  }
}

/* kernel_apply_t (solvers.cpp:24-34 dense, :41-44 sparse) */
static void op_apply_t(const kop* op, const double* u, double* out) {
  if (op->sk) {
    spko_spmv_t(op->sk, u, out);
    return;
  }
  const int64_t n = op->n;
  for (int64_t j = 0; j < n; ++j) out[j] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double ui = u[i];
    if (ui == 0.0) continue;
    const double* row = op->K + i * n;
    for (int64_t j = 0; j < n; ++j) out[j] += row[j] * ui;
  }
}

/* kernel_log_apply (solvers.cpp:52-71 dense, :96-113 sparse) */
static void op_log_apply(const kop* op, const double* lv, double* out) {
  const int64_t n = op->n;
  for (int64_t i = 0; i < n; ++i) {
    double mx = -INFINITY;
    if (op->sk) {
      const spko_csr* M = op->sk;
      for (int64_t p = M->row_ptr[i]; p < M->row_ptr[i + 1]; ++p) {
        if (lv[M->col_idx[p]] == -INFINITY) continue;
        const double t = log(M->values[p]) + lv[M->col_idx[p]];
        mx = mx > t ? mx : t; /* std::max(mx, t) */
      }
      out[i] = -INFINITY;
      if (mx == -INFINITY) continue;
      double acc = 0.0;
      for (int64_t p = M->row_ptr[i]; p < M->row_ptr[i + 1]; ++p) {
        if (lv[M->col_idx[p]] == -INFINITY) continue;
        acc += exp(log(M->values[p]) + lv[M->col_idx[p]] - mx);
      }
      out[i] = mx + log(acc);
    } else {
      const double* row = op->K + i * n;
      for (int64_t j = 0; j < n; ++j) {
        if (row[j] == 0.0 || lv[j] == -INFINITY) continue;
        const double t = log(row[j]) + lv[j];
        mx = mx > t ? mx : t;
      }
      out[i] = -INFINITY;
      if (mx == -INFINITY) continue;
      double acc = 0.0;
      for (int64_t j = 0; j < n; ++j) {
        if (row[j] == 0.0 || lv[j] == -INFINITY) continue;
        acc += exp(log(row[j]) + lv[j] - mx);
      }
      out[i] = mx + log(acc);
    }
  }
}

/* kernel_log_apply_t (solvers.cpp:73-94 dense, :115-136 sparse) */
static void op_log_apply_t(const kop* op, const double* lu, double* out) {
  const int64_t n = op->n;
  double* mx = (double*)malloc(sizeof(double) * n);
  double* acc = (double*)malloc(sizeof(double) * n);
  for (int64_t j = 0; j < n; ++j) {
    mx[j] = -INFINITY;
    acc[j] = 0.0;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (lu[i] == -INFINITY) continue;
    if (op->sk) {
      const spko_csr* M = op->sk;
      for (int64_t p = M->row_ptr[i]; p < M->row_ptr[i + 1]; ++p) {
        const int64_t j = M->col_idx[p];
        const double t = log(M->values[p]) + lu[i];
        mx[j] = mx[j] > t ? mx[j] : t;
      }
    } else {
      const double* row = op->K + i * n;
      for (int64_t j = 0; j < n; ++j)
        if (row[j] > 0.0) {
          const double t = log(row[j]) + lu[i];
          mx[j] = mx[j] > t ? mx[j] : t;
        }
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    if (lu[i] == -INFINITY) continue;
    if (op->sk) {
      const spko_csr* M = op->sk;
      for (int64_t p = M->row_ptr[i]; p < M->row_ptr[i + 1]; ++p) {
        const int64_t j = M->col_idx[p];
        acc[j] += exp(log(M->values[p]) + lu[i] - mx[j]);
      }
    } else {
      const double* row = op->K + i * n;
      for (int64_t j = 0; j < n; ++j)
        if (row[j] > 0.0) acc[j] += exp(log(row[j]) + lu[i] - mx[j]);
    }
  }
  for (int64_t j = 0; j < n; ++j) out[j] = mx[j] != -INFINITY ? mx[j] + log(acc[j]) : -INFINITY;
  free(mx);
  free(acc);
}

/* kernel_coverage (solvers.cpp:138-163) */
static void op_coverage(const kop* op, char* rne, char* cne) {
  const int64_t n = op->n;
  memset(rne, 0, (size_t)n);
  memset(cne, 0, (size_t)n);
  if (op->sk) {
    const spko_csr* M = op->sk;
    for (int64_t i = 0; i < n; ++i) {
      if (M->row_ptr[i + 1] > M->row_ptr[i]) rne[i] = 1;
      for (int64_t p = M->row_ptr[i]; p < M->row_ptr[i + 1]; ++p) cne[M->col_idx[p]] = 1;
    }
  } else {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j)
        if (op->K[i * n + j] > 0.0) {
          rne[i] = 1;
          cne[j] = 1;
        }
  }
}

/* kernel_mean (solvers.cpp:165-177) */
static double op_kernel_mean(const kop* op) {
  double acc = 0.0;
  if (op->sk) {
    for (int64_t p = 0; p < op->sk->nnz; ++p) acc += op->sk->values[p];
  } else {
    for (int64_t k = 0; k < op->n * op->n; ++k) acc += op->K[k];
  }
  const double nd = (double)op->n;
  return acc / (nd * nd);
}

/* TransportPlan::for_each_entry (solvers.hpp:234-252) feeding the row and
 * column marginals (solvers.cpp:215-225) and, when C/coords are given,
 * transport_and_entropy (solvers.cpp:265-276). */
typedef struct {
  const double *u, *v, *lu, *lv;
  int log_domain;
} plan_view;

static inline double plan_t(const plan_view* pv, int64_t i, int64_t j, double kij) {
  if (pv->log_domain) {
    if (pv->lu[i] == -INFINITY || pv->lv[j] == -INFINITY) return 0.0;
    return exp(pv->lu[i] + log(kij) + pv->lv[j]);
  }
  return pv->u[i] * kij * pv->v[j];
}

static void plan_marginals(const kop* op, const plan_view* pv, double* row_m, double* col_m) {
  const int64_t n = op->n;
  for (int64_t k = 0; k < n; ++k) row_m[k] = col_m[k] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (op->sk) {
      for (int64_t p = op->sk->row_ptr[i]; p < op->sk->row_ptr[i + 1]; ++p) {
        const int64_t j = op->sk->col_idx[p];
        const double t = plan_t(pv, i, j, op->sk->values[p]);
        if (t > 0.0) {
          row_m[i] += t;
          col_m[j] += t;
        }
      }
    } else {
      for (int64_t j = 0; j < n; ++j) {
        const double kij = op->K[i * n + j];
        if (!(kij > 0.0)) continue;
        const double t = plan_t(pv, i, j, kij);
        if (t > 0.0) {
          row_m[i] += t;
          col_m[j] += t;
        }
      }
    }
  }
}

static int check_sizes_loop(int64_t n, int64_t na, int64_t nb) {
  return (na != n || nb != n) ? SPKO_E_LENGTH_MISMATCH : SPKO_OK;
}

/* detail::scaling_loop (solvers.hpp:256-395) */
static int scaling_loop(const kop* op, const double* a, const double* b, const spko_cfg* cfg,
                        int policy, double exponent, double* u_out, double* v_out,
                        spko_result* res, char* msg, size_t len) {
  const int64_t n = op->n;
  char* row_ne = (char*)malloc((size_t)n);
  char* col_ne = (char*)malloc((size_t)n);
  op_coverage(op, row_ne, col_ne);
  int64_t masked_rows = 0, masked_cols = 0;
  for (int64_t i = 0; i < n; ++i) masked_rows += row_ne[i] ? 0 : 1;
  for (int64_t j = 0; j < n; ++j) masked_cols += col_ne[j] ? 0 : 1;
  int rc = SPKO_OK;
  double *u = NULL, *v = NULL, *up = NULL, *vp = NULL, *tmp = NULL;
  if ((masked_rows || masked_cols) && policy == SPKO_POLICY_ERROR) {
    char buf[160];
    snprintf(buf, sizeof buf, "kernel has %lld empty rows and %lld empty columns",
             (long long)masked_rows, (long long)masked_cols);
    set_msg(msg, len, "ZeroDenominator", buf);
    rc = SPKO_E_ZERO_DENOMINATOR;
    goto done;
  }
  if (masked_rows == n || masked_cols == n) {
    set_msg(msg, len, "DegenerateSketchError", "kernel has no entries at all");
    rc = SPKO_E_DEGENERATE_SKETCH;
    goto done;
  }
  u = (double*)malloc(sizeof(double) * n);
  v = (double*)malloc(sizeof(double) * n);
  up = (double*)malloc(sizeof(double) * n);
  vp = (double*)malloc(sizeof(double) * n);
  tmp = (double*)malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) u[i] = row_ne[i] ? 1.0 : 0.0;
  for (int64_t j = 0; j < n; ++j) v[j] = col_ne[j] ? 1.0 : 0.0;

  int converged = 0, diverged = 0;
  int64_t t = 0;
  while (t < cfg->max_iter) {
    ++t;
    memcpy(up, u, sizeof(double) * n);
    memcpy(vp, v, sizeof(double) * n);

    op_apply(op, v, tmp);
    for (int64_t i = 0; i < n; ++i) {
      if (!row_ne[i]) continue;
      if (tmp[i] <= 0.0 || !isfinite(tmp[i])) {
        if (policy == SPKO_POLICY_MASK && tmp[i] == 0.0) {
          row_ne[i] = 0;
          u[i] = 0.0;
          ++masked_rows;
          continue;
        }
        if (policy == SPKO_POLICY_MASK) {
          diverged = 1;
          break;
        }
        char buf[160];
        snprintf(buf, sizeof buf, "Kv underflowed at row %lld; consider SolverConfig::stabilize",
                 (long long)i);
        set_msg(msg, len, "ZeroDenominator", buf);
        rc = SPKO_E_ZERO_DENOMINATOR;
        goto done;
      }
      const double q = a[i] / tmp[i];
      u[i] = (exponent == 1.0) ? q : pow(q, exponent);
      if (!(u[i] <= 1e150) && policy == SPKO_POLICY_MASK) {
        diverged = 1;
        break;
      }
    }
    if (diverged) {
      memcpy(u, up, sizeof(double) * n);
      memcpy(v, vp, sizeof(double) * n);
      break;
    }

    op_apply_t(op, u, tmp);
    for (int64_t j = 0; j < n; ++j) {
      if (!col_ne[j]) continue;
      if (tmp[j] <= 0.0 || !isfinite(tmp[j])) {
        if (policy == SPKO_POLICY_MASK && tmp[j] == 0.0) {
          col_ne[j] = 0;
          v[j] = 0.0;
          ++masked_cols;
          continue;
        }
        if (policy == SPKO_POLICY_MASK) {
          diverged = 1;
          break;
        }
        char buf[160];
        snprintf(buf, sizeof buf,
                 "K'u underflowed at column %lld; consider SolverConfig::stabilize", (long long)j);
        set_msg(msg, len, "ZeroDenominator", buf);
        rc = SPKO_E_ZERO_DENOMINATOR;
        goto done;
      }
      const double q = b[j] / tmp[j];
      v[j] = (exponent == 1.0) ? q : pow(q, exponent);
      if (!(v[j] <= 1e150) && policy == SPKO_POLICY_MASK) {
        diverged = 1;
        break;
      }
    }
    if (diverged) {
      memcpy(u, up, sizeof(double) * n);
      memcpy(v, vp, sizeof(double) * n);
      break;
    }
    if (masked_rows == n || masked_cols == n) {
      set_msg(msg, len, "DegenerateSketchError", "masking removed every atom");
      rc = SPKO_E_DEGENERATE_SKETCH;
      goto done;
    }
    if (t >= 2) {
      double err = 0.0;
      for (int64_t i = 0; i < n; ++i) err += fabs(u[i] - up[i]);
      for (int64_t j = 0; j < n; ++j) err += fabs(v[j] - vp[j]);
      if (err <= cfg->delta) {
        converged = 1;
        break;
      }
    }
  }
  {
    plan_view pv = {u, v, NULL, NULL, 0};
    double* row_m = (double*)malloc(sizeof(double) * n);
    double* col_m = (double*)malloc(sizeof(double) * n);
    plan_marginals(op, &pv, row_m, col_m);
    double rr = 0.0, rcc = 0.0;
    for (int64_t i = 0; i < n; ++i) rr += fabs(row_m[i] - a[i]);
    for (int64_t j = 0; j < n; ++j) rcc += fabs(col_m[j] - b[j]);
    free(row_m);
    free(col_m);
    res->iterations = t;
    res->converged = converged;
    res->diverged = diverged;
    res->log_domain = 0;
    res->masked_rows = masked_rows;
    res->masked_cols = masked_cols;
    res->residual_row = rr;
    res->residual_col = rcc;
    res->kernel_mean = op_kernel_mean(op);
    memcpy(u_out, u, sizeof(double) * n);
    memcpy(v_out, v, sizeof(double) * n);
  }
done:
  free(row_ne);
  free(col_ne);
  free(u);
  free(v);
  free(up);
  free(vp);
  free(tmp);
  return rc;
}

/* detail::log_scaling_loop (solvers.hpp:397-513) */
static int log_scaling_loop(const kop* op, const double* a, const double* b,
                            const spko_cfg* cfg, int policy, double exponent, double* u_out,
                            double* v_out, double* lu_out, double* lv_out, spko_result* res,
                            char* msg, size_t len) {
  const int64_t n = op->n;
  char* row_ne = (char*)malloc((size_t)n);
  char* col_ne = (char*)malloc((size_t)n);
  op_coverage(op, row_ne, col_ne);
  int64_t masked_rows = 0, masked_cols = 0;
  for (int64_t i = 0; i < n; ++i) masked_rows += row_ne[i] ? 0 : 1;
  for (int64_t j = 0; j < n; ++j) masked_cols += col_ne[j] ? 0 : 1;
  int rc = SPKO_OK;
  double *lu = NULL, *lv = NULL, *lup = NULL, *lvp = NULL, *tmp = NULL, *la = NULL, *lb = NULL;
  if ((masked_rows || masked_cols) && policy == SPKO_POLICY_ERROR) {
    set_msg(msg, len, "ZeroDenominator", "kernel has empty rows or columns");
    rc = SPKO_E_ZERO_DENOMINATOR;
    goto done;
  }
  if (masked_rows == n || masked_cols == n) {
    set_msg(msg, len, "DegenerateSketchError", "kernel has no entries at all");
    rc = SPKO_E_DEGENERATE_SKETCH;
    goto done;
  }
  la = (double*)malloc(sizeof(double) * n);
  lb = (double*)malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) la[i] = a[i] > 0.0 ? log(a[i]) : -INFINITY;
  for (int64_t j = 0; j < n; ++j) lb[j] = b[j] > 0.0 ? log(b[j]) : -INFINITY;
  lu = (double*)malloc(sizeof(double) * n);
  lv = (double*)malloc(sizeof(double) * n);
  lup = (double*)malloc(sizeof(double) * n);
  lvp = (double*)malloc(sizeof(double) * n);
  tmp = (double*)malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) lu[i] = row_ne[i] ? 0.0 : -INFINITY;
  for (int64_t j = 0; j < n; ++j) lv[j] = col_ne[j] ? 0.0 : -INFINITY;

  int converged = 0;
  int64_t t = 0;
  while (t < cfg->max_iter) {
    ++t;
    memcpy(lup, lu, sizeof(double) * n);
    memcpy(lvp, lv, sizeof(double) * n);
    op_log_apply(op, lv, tmp);
    for (int64_t i = 0; i < n; ++i) {
      if (!row_ne[i]) continue;
      if (tmp[i] == -INFINITY) {
        if (policy == SPKO_POLICY_MASK) {
          row_ne[i] = 0;
          lu[i] = -INFINITY;
          ++masked_rows;
          continue;
        }
        char buf[96];
        snprintf(buf, sizeof buf, "Kv vanished at row %lld", (long long)i);
        set_msg(msg, len, "ZeroDenominator", buf);
        rc = SPKO_E_ZERO_DENOMINATOR;
        goto done;
      }
      lu[i] = exponent * (la[i] - tmp[i]);
    }
    op_log_apply_t(op, lu, tmp);
    for (int64_t j = 0; j < n; ++j) {
      if (!col_ne[j]) continue;
      if (tmp[j] == -INFINITY) {
        if (policy == SPKO_POLICY_MASK) {
          col_ne[j] = 0;
          lv[j] = -INFINITY;
          ++masked_cols;
          continue;
        }
        char buf[96];
        snprintf(buf, sizeof buf, "K'u vanished at column %lld", (long long)j);
        set_msg(msg, len, "ZeroDenominator", buf);
        rc = SPKO_E_ZERO_DENOMINATOR;
        goto done;
      }
      lv[j] = exponent * (lb[j] - tmp[j]);
    }
    if (masked_rows == n || masked_cols == n) {
      set_msg(msg, len, "DegenerateSketchError", "masking removed every atom");
      rc = SPKO_E_DEGENERATE_SKETCH;
      goto done;
    }
    if (t >= 2) {
      double err = 0.0;
      for (int64_t i = 0; i < n; ++i)
        if (row_ne[i]) err += fabs(lu[i] - lup[i]);
      for (int64_t j = 0; j < n; ++j)
        if (col_ne[j]) err += fabs(lv[j] - lvp[j]);
      if (err <= cfg->delta) {
        converged = 1;
        break;
      }
    }
  }
  {
    double* u = (double*)malloc(sizeof(double) * n);
    double* v = (double*)malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) u[i] = exp(lu[i]);
    for (int64_t j = 0; j < n; ++j) v[j] = exp(lv[j]);
    plan_view pv = {u, v, lu, lv, 1};
    double* row_m = (double*)malloc(sizeof(double) * n);
    double* col_m = (double*)malloc(sizeof(double) * n);
    plan_marginals(op, &pv, row_m, col_m);
    double rr = 0.0, rcc = 0.0;
    for (int64_t i = 0; i < n; ++i) rr += fabs(row_m[i] - a[i]);
    for (int64_t j = 0; j < n; ++j) rcc += fabs(col_m[j] - b[j]);
    free(row_m);
    free(col_m);
    res->iterations = t;
    res->converged = converged;
    res->diverged = 0;
    res->log_domain = 1;
    res->masked_rows = masked_rows;
    res->masked_cols = masked_cols;
    res->residual_row = rr;
    res->residual_col = rcc;
    res->kernel_mean = op_kernel_mean(op);
    memcpy(u_out, u, sizeof(double) * n);
    memcpy(v_out, v, sizeof(double) * n);
    if (lu_out) memcpy(lu_out, lu, sizeof(double) * n);
    if (lv_out) memcpy(lv_out, lv, sizeof(double) * n);
    free(u);
    free(v);
  }
done:
  free(row_ne);
  free(col_ne);
  free(la);
  free(lb);
  free(lu);
  free(lv);
  free(lup);
  free(lvp);
  free(tmp);
  return rc;
}

/* sinkhorn_ot / sinkhorn_uot (solvers.hpp:209-232) */
int spko_sinkhorn(const spko_csr* sk, const double* K, int64_t n, const double* a,
                  const double* b, double a_total, double b_total, const spko_cfg* cfg,
                  int policy, int uot, double* u, double* v, double* log_u, double* log_v,
                  spko_result* res, char* msg, size_t len) {
  double f = 1.0;
  if (!uot) {
    if (fabs(a_total - 1.0) > 1e-8 || fabs(b_total - 1.0) > 1e-8) {
      set_msg(msg, len, "NotNormalized", "sinkhorn_ot requires simplex inputs");
      return SPKO_E_NOT_NORMALIZED;
    }
  } else {
    if (!(cfg->lambda > 0) || !isfinite(cfg->lambda)) {
      set_msg(msg, len, NULL, "sinkhorn_uot needs finite lambda > 0");
      return SPKO_E_ERROR;
    }
    f = cfg->lambda / (cfg->lambda + cfg->epsilon);
  }
  kop op = {sk, K, sk ? sk->n : n};
  if (check_sizes_loop(op.n, n, n) != SPKO_OK) return SPKO_E_LENGTH_MISMATCH;
  if (cfg->stabilize)
    return log_scaling_loop(&op, a, b, cfg, policy, f, u, v, log_u, log_v, res, msg, len);
  return scaling_loop(&op, a, b, cfg, policy, f, u, v, res, msg, len);
}

/* time_scaling_iters (harness.cpp:262-278) */
double spko_time_scaling_iters(const spko_csr* sk, const double* a, const double* b,
                               int64_t iters, double* u, double* v) {
  const int64_t n = sk->n;
  double* tmp = (double*)malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) u[i] = v[i] = 1.0;
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int64_t t = 0; t < iters; ++t) {
    spko_spmv(sk, v, tmp);
    for (int64_t i = 0; i < n; ++i) u[i] = tmp[i] > 0.0 ? a[i] / tmp[i] : 0.0;
    spko_spmv_t(sk, u, tmp);
    for (int64_t j = 0; j < n; ++j) v[j] = tmp[j] > 0.0 ? b[j] / tmp[j] : 0.0;
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  free(tmp);
  const double dt = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  return dt / (double)iters;
}

/* kl_divergence (solvers.cpp:246-260) */
int spko_kl_divergence(const double* x, const double* y, int64_t n, double* out) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (x[i] > 0.0) {
      if (y[i] <= 0.0) return SPKO_E_ERROR;
      acc += x[i] * log(x[i] / y[i]) - x[i] + y[i];
    } else {
      acc += y[i];
    }
  }
  *out = acc;
  return SPKO_OK;
}

/* transport_and_entropy + ot_objective / uot_objective + marginals
 * (solvers.cpp:215-225, 265-293). */
int spko_readout(const spko_csr* sk, const double* K, int64_t n, const double* u,
                 const double* v, const double* log_u, const double* log_v, int log_domain,
                 const double* C, const double* x, const double* y, int dim, int cost_kind,
                 double eta, double scale, const double* a, const double* b, int uot,
                 double lambda, double eps, double* row_m, double* col_m, double* objective,
                 char* msg, size_t len) {
  kop op = {sk, K, sk ? sk->n : n};
  plan_view pv = {u, v, log_u, log_v, log_domain};
  double cost = 0.0, entropy = 0.0;
  const int have_cost = (C != NULL) || (x != NULL && y != NULL);
  for (int64_t i = 0; i < op.n && have_cost; ++i) {
    int64_t pb = 0, pe = op.n;
    if (sk) {
      pb = sk->row_ptr[i];
      pe = sk->row_ptr[i + 1];
    }
    for (int64_t p = pb; p < pe; ++p) {
      const int64_t j = sk ? (int64_t)sk->col_idx[p] : p;
      const double kij = sk ? sk->values[p] : K[i * op.n + j];
      if (!sk && !(kij > 0.0)) continue;
      const double t = plan_t(&pv, i, j, kij);
      if (!(t > 0.0)) continue;
      double cij;
      if (C) {
        cij = C[i * op.n + j];
      } else {
        cij = spko_cost_entry(x + i * dim, y + j * dim, dim, cost_kind, eta) / scale;
      }
      if (isinf(cij)) {
        set_msg(msg, len, "InfiniteCostOnSupport", "plan mass on a blocked entry");
        return SPKO_E_INFINITE_COST_ON_SUPPORT;
      }
      cost += t * cij;
      entropy -= t * (log(t) - 1.0);
    }
  }
  double* rm = row_m ? row_m : (double*)malloc(sizeof(double) * op.n);
  double* cm = col_m ? col_m : (double*)malloc(sizeof(double) * op.n);
  plan_marginals(&op, &pv, rm, cm);
  int rc = SPKO_OK;
  if (objective && have_cost) {
    if (!uot) {
      *objective = cost - eps * entropy;
    } else {
      double kl_a = 0.0, kl_b = 0.0;
      rc = spko_kl_divergence(rm, a, op.n, &kl_a);
      if (rc == SPKO_OK) rc = spko_kl_divergence(cm, b, op.n, &kl_b);
      if (rc != SPKO_OK) set_msg(msg, len, NULL, "KL undefined: mass off support");
      *objective = cost + lambda * kl_a + lambda * kl_b - eps * entropy;
    }
  }
  if (!row_m) free(rm);
  if (!col_m) free(cm);
  return rc;
}

/* build_sketch + spar_sink_ot/uot (solvers.cpp:314-378) */
int spko_spar_sink(const double* K, double nnz_ratio, const double* C, int64_t n,
                   const double* a, const double* b, double a_total, double b_total,
                   const spko_cfg* cfg, double s, uint64_t seed, double theta, int probs,
                   int strict, int uot, double* u, double* v, double* log_u, double* log_v,
                   spko_result* res, double* objective, int64_t* sketch_nnz, spko_csr* sk_out,
                   char* msg, size_t len) {
  spko_plan plan;
  memset(&plan, 0, sizeof plan);
  int rc;
  if (probs == 1)
    rc = spko_uniform_probabilities(n, K, nnz_ratio, &plan);
  else if (uot)
    rc = spko_uot_probabilities(a, b, n, K, nnz_ratio, cfg->lambda, cfg->epsilon, &plan);
  else
    rc = spko_ot_probabilities(a, b, n, K, nnz_ratio, &plan);
  if (rc != SPKO_OK) return rc;
  if (theta > 0.0) {
    rc = spko_shrink_with_uniform(&plan, theta);
    if (rc != SPKO_OK) {
      spko_plan_free(&plan);
      return rc;
    }
  }
  spko_csr sk;
  memset(&sk, 0, sizeof sk);
  rc = spko_poisson_sparsify(K, n, &plan, s, seed, &sk);
  spko_plan_free(&plan);
  if (rc != SPKO_OK) return rc;
  if (strict) {
    char* rne = (char*)malloc((size_t)n);
    char* cne = (char*)malloc((size_t)n);
    kop op = {&sk, NULL, n};
    op_coverage(&op, rne, cne);
    for (int64_t i = 0; i < n; ++i)
      if (!rne[i] || !cne[i]) {
        char buf[160];
        snprintf(buf, sizeof buf,
                 "sketch orphaned atom %lld; raise s or theta, or use a different seed",
                 (long long)i);
        set_msg(msg, len, "DegenerateSketchError", buf);
        rc = SPKO_E_DEGENERATE_SKETCH;
        break;
      }
    free(rne);
    free(cne);
    if (rc != SPKO_OK) {
      spko_csr_free(&sk);
      return rc;
    }
  }
  double* lu = log_u ? log_u : (double*)malloc(sizeof(double) * n);
  double* lv = log_v ? log_v : (double*)malloc(sizeof(double) * n);
  rc = spko_sinkhorn(&sk, NULL, n, a, b, a_total, b_total, cfg,
                     strict ? SPKO_POLICY_ERROR : SPKO_POLICY_MASK, uot, u, v, lu, lv, res,
                     msg, len);
  if (rc == SPKO_OK) {
    rc = spko_readout(&sk, NULL, n, u, v, lu, lv, res->log_domain, C, NULL, NULL, 0, 0,
                      0.0, 1.0, a, b, uot, cfg->lambda, cfg->epsilon, NULL, NULL, objective, msg,
                      len);
    *sketch_nnz = sk.nnz;
  }
  if (!log_u) free(lu);
  if (!log_v) free(lv);
  if (sk_out && rc == SPKO_OK)
    *sk_out = sk;
  else
    spko_csr_free(&sk);
  return rc;
}
