// ref_capi.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE / CPU BASELINE ONLY. oracle/Makefile compiles this file
// together with /root/reference/proj/src/*.cpp (never copied) into
// oracle/_ref/libsparsink_ref.so. Tests use it to pin the C restatement
// (oracle/spk_oracle.c) to the reference bit-for-bit; bench.py --impl
// reference uses it to time the reference's own CPU path.
//
// Every function below only marshals plain arrays into the reference's
// public types and calls the reference's public API (proj/include/sparsink).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <iostream>  // std::ios_base::Init for the statically linked libstdc++ (ofstream writers)
#include <limits>
#include <string>
#include <vector>

#include "sparsink/errors.hpp"
#include "sparsink/geometry.hpp"
#include "sparsink/harness.hpp"
#include "sparsink/barycenter.hpp"
#include "sparsink/measures.hpp"
#include "sparsink/rng.hpp"
#include "sparsink/solvers.hpp"
#include "sparsink/sparsify.hpp"

using namespace sparsink;

namespace {

// Same numbering as include/spk.h SPK_E_*.
int kind_of(const Error& e) {
#define K(cls, code) \
  if (dynamic_cast<const cls*>(&e)) return code;
  K(NegativeWeight, 2) K(LengthMismatch, 3) K(NotNormalized, 4) K(AllBlack, 5)
  K(EmptyOutput, 6) K(DimensionMismatch, 7) K(NonPositiveEta, 8) K(NonPositiveEpsilon, 9)
  K(DegenerateSupport, 10) K(AllZeroKernel, 11) K(ThetaOutOfRange, 12) K(BudgetTooLarge, 13)
  K(EmptyWindow, 14) K(InfiniteCostOnSupport, 15) K(IoError, 16) K(ZeroDenominator, 17)
  K(BaselineFailed, 18) K(DegenerateSketchError, 19)
#undef K
  return 1;
}

thread_local std::string g_msg;
thread_local int g_category = 0;

template <class F>
int guard(F&& f) {
  try {
    f();
    g_msg.clear();
    g_category = 0;
    return 0;
  } catch (const Error& e) {
    g_msg = e.what();
    g_category = static_cast<int>(e.category());
    return kind_of(e);
  } catch (const std::exception& e) {
    g_msg = e.what();
    g_category = 5;
    return 99;
  }
}

PointList points(const double* x, int64_t n, int dim) {
  PointList p;
  p.dim = static_cast<std::size_t>(dim);
  p.coords.assign(x, x + n * dim);
  return p;
}

DiscreteMeasure measure(const double* w, int64_t n) {
  // Support is irrelevant to the solvers; give each atom a 1-D coordinate.
  PointList sup;
  sup.dim = 1;
  sup.coords.resize(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) sup.coords[i] = static_cast<double>(i);
  return new_measure(std::vector<double>(w, w + n), std::move(sup), false);
}

KernelMatrix kernel(const double* K, int64_t n, double eps, double nnz_ratio) {
  KernelMatrix km;
  km.epsilon = eps;
  km.nnz_ratio = nnz_ratio;
  km.entries = Matrix(static_cast<std::size_t>(n), static_cast<std::size_t>(n));
  std::memcpy(km.entries.data().data(), K, sizeof(double) * n * n);
  return km;
}

CostMatrix cost(const double* C, int64_t n) {
  CostMatrix cm;
  cm.entries = Matrix(static_cast<std::size_t>(n), static_cast<std::size_t>(n));
  std::memcpy(cm.entries.data().data(), C, sizeof(double) * n * n);
  return cm;
}

SparseKernel sketch(int64_t n, const int64_t* rp, const uint32_t* ci, const double* val) {
  SparseKernel sk;
  sk.n = static_cast<std::size_t>(n);
  sk.row_ptr.assign(rp, rp + n + 1);
  const int64_t nnz = rp[n];
  sk.col_idx.assign(ci, ci + nnz);
  sk.values.assign(val, val + nnz);
  sk.realized_nnz = static_cast<std::size_t>(nnz);
  return sk;
}

SamplingPlan make_plan(int kind, const double* a, const double* b, int64_t n,
                       const KernelMatrix& K, double lambda, double eps, double theta) {
  auto da = measure(a, n), db = measure(b, n);
  SamplingPlan plan = kind == 3   ? uniform_probabilities(K)
                      : kind == 1 ? uot_probabilities(da, db, K, lambda, eps)
                                  : ot_probabilities(da, db, K);
  if (theta > 0.0) plan = shrink_with_uniform(plan, theta);
  return plan;
}

struct ref_result {
  int64_t iterations;
  int32_t converged, diverged, log_domain, pad;
  int64_t masked_rows, masked_cols;
  double residual_row, residual_col, kernel_mean, objective, wall_time_s;
  int64_t sketch_nnz;
};

void fill(ref_result* r, const SolveResult& s) {
  r->iterations = static_cast<int64_t>(s.report.iterations);
  r->converged = s.report.converged;
  r->diverged = s.report.diverged;
  r->log_domain = s.plan.log_domain;
  r->masked_rows = static_cast<int64_t>(s.plan.masked_rows);
  r->masked_cols = static_cast<int64_t>(s.plan.masked_cols);
  r->residual_row = s.report.marginal_residual_row;
  r->residual_col = s.report.marginal_residual_col;
  r->kernel_mean = s.report.kernel_mean;
  r->objective = s.report.objective;
  r->wall_time_s = s.report.wall_time_s;
  r->sketch_nnz = s.report.sketch_nnz ? static_cast<int64_t>(*s.report.sketch_nnz) : -1;
}

void copy_out(const SolveResult& s, double* u, double* v, double* lu, double* lv) {
  std::memcpy(u, s.plan.u.data(), sizeof(double) * s.plan.u.size());
  std::memcpy(v, s.plan.v.data(), sizeof(double) * s.plan.v.size());
  if (s.plan.log_domain) {
    if (lu) std::memcpy(lu, s.plan.log_u.data(), sizeof(double) * s.plan.log_u.size());
    if (lv) std::memcpy(lv, s.plan.log_v.data(), sizeof(double) * s.plan.log_v.size());
  }
}

SolverConfig config(double eps, double lambda, double delta, int64_t max_iter, int stabilize) {
  SolverConfig cfg;
  cfg.epsilon = eps;
  cfg.lambda = lambda;
  cfg.delta = delta;
  cfg.max_iter = static_cast<std::size_t>(max_iter);
  cfg.stabilize = stabilize != 0;
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error(int* category) {
  if (category) *category = g_category;
  return g_msg.c_str();
}

void ref_free(void* p) { std::free(p); }

uint64_t ref_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

void ref_rng_doubles(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  CounterRng rng(seed, stream);
  for (int64_t k = 0; k < count; ++k) out[k] = rng.next_double();
}

void ref_rng_normals(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  CounterRng rng(seed, stream);
  for (int64_t k = 0; k < count; ++k) out[k] = rng.next_normal();
}

// geometry.hpp:28-34
int ref_pairwise_cost(const double* x, int64_t nx, const double* y, int64_t ny, int dim,
                      int kind, double eta, double* C, double* c0) {
  return guard([&] {
    auto px = points(x, nx, dim), py = points(y, ny, dim);
    CostMatrix cm = kind == 2   ? wfr_cost(px, py, eta)
                    : kind == 1 ? euclidean_cost(px, py)
                                : sq_euclidean_cost(px, py);
    std::memcpy(C, cm.entries.data().data(), sizeof(double) * nx * ny);
    *c0 = cm.c0;
  });
}

int ref_kernel_from_cost(const double* C, int64_t n, double eps, double* K, double* nnz_ratio) {
  return guard([&] {
    KernelMatrix km = kernel_from_cost(cost(C, n), eps);
    std::memcpy(K, km.entries.data().data(), sizeof(double) * n * n);
    *nnz_ratio = km.nnz_ratio;
  });
}

// Plan probabilities evaluated on the full grid (sparsify.hpp:74-90).
int ref_plan_probs(int kind, const double* a, const double* b, int64_t n, const double* K,
                   double nnz_ratio, double lambda, double eps, double theta, double* probs,
                   int* factorized) {
  return guard([&] {
    auto km = kernel(K, n, eps, nnz_ratio);
    auto plan = make_plan(kind, a, b, n, km, lambda, eps, theta);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) probs[i * n + j] = plan.prob(i, j);
    *factorized = plan.factorized_storage();
  });
}

// poisson_sparsify (sparsify.hpp:94-95). Output arrays malloc'd; free with ref_free.
int ref_poisson_sparsify(int kind, const double* a, const double* b, int64_t n, const double* K,
                         double nnz_ratio, double lambda, double eps, double theta, double s,
                         uint64_t seed, int64_t** row_ptr, uint32_t** col_idx, double** values,
                         int64_t* nnz) {
  return guard([&] {
    auto km = kernel(K, n, eps, nnz_ratio);
    auto plan = make_plan(kind, a, b, n, km, lambda, eps, theta);
    SparseKernel sk = poisson_sparsify(km, plan, s, seed);
    const std::size_t m = sk.values.size();
    *nnz = static_cast<int64_t>(m);
    *row_ptr = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (n + 1)));
    *col_idx = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * (m + 1)));
    *values = static_cast<double*>(std::malloc(sizeof(double) * (m + 1)));
    for (int64_t i = 0; i <= n; ++i) (*row_ptr)[i] = static_cast<int64_t>(sk.row_ptr[i]);
    std::memcpy(*col_idx, sk.col_idx.data(), sizeof(uint32_t) * m);
    std::memcpy(*values, sk.values.data(), sizeof(double) * m);
  });
}

// spmv / spmv_t (sparsify.hpp:97-98)
int ref_spmv(int64_t n, const int64_t* rp, const uint32_t* ci, const double* val, const double* x,
             int transpose, double* out) {
  return guard([&] {
    auto sk = sketch(n, rp, ci, val);
    std::vector<double> xv(x, x + n);
    auto y = transpose ? spmv_t(sk, xv) : spmv(sk, xv);
    std::memcpy(out, y.data(), sizeof(double) * n);
  });
}

// sinkhorn_ot / sinkhorn_uot on a sketch (rp != NULL) or dense K
// (solvers.hpp:137-147), policy 0 = Error, 1 = Mask.
int ref_sinkhorn(int64_t n, const int64_t* rp, const uint32_t* ci, const double* val,
                 const double* K, double nnz_ratio, const double* a, const double* b, double eps,
                 double lambda, double delta, int64_t max_iter, int stabilize, int policy, int uot,
                 double* u, double* v, double* lu, double* lv, ref_result* res) {
  return guard([&] {
    auto da = measure(a, n), db = measure(b, n);
    auto cfg = config(eps, lambda, delta, max_iter, stabilize);
    const EmptyPolicy pol = policy ? EmptyPolicy::Mask : EmptyPolicy::Error;
    SolveResult r;
    if (rp) {
      auto sk = sketch(n, rp, ci, val);
      r = uot ? sinkhorn_uot(sk, da, db, cfg, pol) : sinkhorn_ot(sk, da, db, cfg, pol);
    } else {
      auto km = kernel(K, n, eps, nnz_ratio);
      r = uot ? sinkhorn_uot(km, da, db, cfg, pol) : sinkhorn_ot(km, da, db, cfg, pol);
    }
    fill(res, r);
    copy_out(r, u, v, lu, lv);
  });
}

// spar_sink_ot / spar_sink_uot (solvers.hpp:159-167) on dense K and C.
int ref_spar_sink(int64_t n, const double* K, double nnz_ratio, const double* C, const double* a,
                  const double* b, double eps, double lambda, double delta, int64_t max_iter,
                  int stabilize, double s, uint64_t seed, double theta, int probs, int strict,
                  int uot, double* u, double* v, double* lu, double* lv, ref_result* res) {
  return guard([&] {
    auto da = measure(a, n), db = measure(b, n);
    auto cfg = config(eps, lambda, delta, max_iter, stabilize);
    auto km = kernel(K, n, eps, nnz_ratio);
    auto cm = cost(C, n);
    SparSinkOptions opts;
    opts.theta = theta;
    opts.probs = probs ? SketchProbs::Uniform : SketchProbs::Importance;
    opts.strict = strict != 0;
    SolveResult r = uot ? spar_sink_uot(km, cm, da, db, cfg, s, seed, opts)
                        : spar_sink_ot(km, cm, da, db, cfg, s, seed, opts);
    fill(res, r);
    copy_out(r, u, v, lu, lv);
  });
}

// Objective readout on a sketch (ot_objective / uot_objective,
// solvers.hpp:170-177) plus the plan marginals (TransportPlan::row_marginal,
// col_marginal).
int ref_readout(int64_t n, const int64_t* rp, const uint32_t* ci, const double* val,
                const double* u, const double* v, const double* lu, const double* lv,
                int log_domain, const double* C, const double* a, const double* b, int uot,
                double lambda, double eps, double* row_m, double* col_m, double* objective) {
  return guard([&] {
    auto sk = sketch(n, rp, ci, val);
    TransportPlan T;
    T.u.assign(u, u + n);
    T.v.assign(v, v + n);
    T.log_domain = log_domain != 0;
    if (log_domain) {
      T.log_u.assign(lu, lu + n);
      T.log_v.assign(lv, lv + n);
    }
    T.sparse_kernel = &sk;
    auto rm = T.row_marginal();
    auto cm = T.col_marginal();
    std::memcpy(row_m, rm.data(), sizeof(double) * n);
    std::memcpy(col_m, cm.data(), sizeof(double) * n);
    auto cc = cost(C, n);
    if (uot) {
      auto da = measure(a, n), db = measure(b, n);
      *objective = uot_objective(T, cc, da, db, lambda, eps);
    } else {
      *objective = ot_objective(T, cc, eps);
    }
  });
}

// The reference's per-iteration timer semantics (harness.cpp:262-278), built
// from its public kernel_apply / kernel_apply_t shims: `iters` bare scaling
// iterations on a sketch. Returns seconds per iteration (steady_clock).
double ref_time_scaling_iters(int64_t n, const int64_t* rp, const uint32_t* ci,
                              const double* val, const double* a, const double* b,
                              int64_t iters, double* u_out, double* v_out) {
  auto sk = sketch(n, rp, ci, val);
  std::vector<double> u(n, 1.0), v(n, 1.0), tmp(n);
  const auto t0 = std::chrono::steady_clock::now();
  for (int64_t t = 0; t < iters; ++t) {
    kernel_apply(sk, v, tmp);
    for (int64_t i = 0; i < n; ++i) u[i] = tmp[i] > 0.0 ? a[i] / tmp[i] : 0.0;
    kernel_apply_t(sk, u, tmp);
    for (int64_t j = 0; j < n; ++j) v[j] = tmp[j] > 0.0 ? b[j] / tmp[j] : 0.0;
  }
  const double dt =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (u_out) std::memcpy(u_out, u.data(), sizeof(double) * n);
  if (v_out) std::memcpy(v_out, v.data(), sizeof(double) * n);
  return dt / static_cast<double>(iters);
}

// sinkhorn_ot<SparseKernel> wall time for `iters` fixed iterations
// (delta = -1 so the t>=2 stop never fires): the reference's own loop.
int ref_sparse_loop_timed_stab(int64_t n, const int64_t* rp, const uint32_t* ci, const double* val,
                               const double* a, const double* b, double eps, double lambda,
                               int64_t iters, int uot, int stabilize, double* seconds, ref_result* res) {
  return guard([&] {
    auto sk = sketch(n, rp, ci, val);
    auto da = measure(a, n), db = measure(b, n);
    auto cfg = config(eps, lambda, -1.0, iters, stabilize);
    const auto t0 = std::chrono::steady_clock::now();
    SolveResult r = uot ? sinkhorn_uot(sk, da, db, cfg, EmptyPolicy::Mask)
                        : sinkhorn_ot(sk, da, db, cfg, EmptyPolicy::Mask);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    fill(res, r);
  });
}

int ref_sparse_loop_timed(int64_t n, const int64_t* rp, const uint32_t* ci, const double* val,
                          const double* a, const double* b, double eps, double lambda,
                          int64_t iters, int uot, double* seconds, ref_result* res) {
  return guard([&] {
    auto sk = sketch(n, rp, ci, val);
    auto da = measure(a, n), db = measure(b, n);
    auto cfg = config(eps, lambda, -1.0, iters, 0);
    const auto t0 = std::chrono::steady_clock::now();
    SolveResult r = uot ? sinkhorn_uot(sk, da, db, cfg, EmptyPolicy::Mask)
                        : sinkhorn_ot(sk, da, db, cfg, EmptyPolicy::Mask);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    fill(res, r);
  });
}


// ---- frame-pair caller: measures.cpp:36-85, harness.cpp:349-437 ----

static FrameImage frame(const double* px, int64_t h, int64_t w) {
  FrameImage f;
  f.height = (std::size_t)h;
  f.width = (std::size_t)w;
  f.pixels.assign(px, px + h * w);
  return f;
}

int ref_measure_from_image(const double* px, int64_t h, int64_t w, double* coords, double* weights) {
  return guard([&] {
    DiscreteMeasure m = measure_from_image(frame(px, h, w));
    std::memcpy(coords, m.support.coords.data(), sizeof(double) * m.support.coords.size());
    std::memcpy(weights, m.weights.data(), sizeof(double) * m.weights.size());
  });
}

int ref_mean_pool(const double* px, int64_t h, int64_t w, int64_t filter, int64_t stride, double* out, int64_t* oh,
                  int64_t* ow) {
  return guard([&] {
    FrameImage o = mean_pool(frame(px, h, w), (std::size_t)filter, (std::size_t)stride);
    *oh = (int64_t)o.height;
    *ow = (int64_t)o.width;
    std::memcpy(out, o.pixels.data(), sizeof(double) * o.pixels.size());
  });
}

int ref_pairwise_wfr(const double* frames, int64_t nframes, int64_t h, int64_t w, double eta, double lambda,
                     double eps, double s_mult, uint64_t seed, int64_t stride, int exact, double* dist, int64_t* m,
                     int64_t* failed) {
  return guard([&] {
    std::vector<FrameImage> fs;
    for (int64_t k = 0; k < nframes; ++k) fs.push_back(frame(frames + k * h * w, h, w));
    PairwiseWfrResult r = pairwise_wfr(fs, eta, lambda, eps, s_mult, seed, (std::size_t)stride, exact != 0);
    *m = (int64_t)r.distances.rows();
    *failed = (int64_t)r.failed_pairs;
    for (int64_t i = 0; i < *m; ++i)
      for (int64_t j = 0; j < *m; ++j) dist[i * *m + j] = r.distances(i, j);
  });
}

int ref_predict_ed(const double* d, int64_t m, int64_t t_es, int64_t lo, int64_t hi, int64_t t_true, int64_t* t_hat,
                   double* err) {
  return guard([&] {
    Matrix dm((std::size_t)m, (std::size_t)m, 0.0);
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < m; ++j) dm(i, j) = d[i * m + j];
    EdPrediction p = predict_ed(dm, (std::size_t)t_es, (std::size_t)lo, (std::size_t)hi, (std::size_t)t_true);
    *t_hat = (int64_t)p.t_ed_hat;
    *err = p.error;
  });
}


// ---- barycenters (barycenter.hpp:48-206, barycenter.cpp:8-40) ----------------------

struct ref_ibp_result {
  int64_t iterations;
  int32_t converged, diverged;
  int64_t masked_atoms;
};

static void fill_ibp(ref_ibp_result* r, const BarycenterResult& b, double* q) {
  r->iterations = (int64_t)b.iterations;
  r->converged = b.converged;
  r->diverged = b.diverged;
  r->masked_atoms = (int64_t)b.masked_atoms;
  std::memcpy(q, b.weights.data(), sizeof(double) * b.weights.size());
}

// ibp<KernelMatrix> (dense) or ibp<SparseKernel> (rp != NULL: m CSR sketches back to back)
int ref_ibp(int32_t m, int64_t n, const double* K, const double* nnz_ratio, const int64_t* rp, const uint32_t* ci,
            const double* val, const int64_t* nnz, const double* b, const double* w, double delta, int64_t max_iter,
            int policy, double* q, ref_ibp_result* res) {
  return guard([&] {
    std::vector<DiscreteMeasure> ms;
    for (int k = 0; k < m; ++k) ms.push_back(measure(b + k * n, n));
    std::vector<const DiscreteMeasure*> mp;
    for (auto& x : ms) mp.push_back(&x);
    BarycenterConfig cfg;
    cfg.delta = delta;
    cfg.max_iter = (std::size_t)max_iter;
    const EmptyPolicy pol = policy ? EmptyPolicy::Mask : EmptyPolicy::Error;
    std::vector<double> wv(w, w + m);
    if (rp) {
      std::vector<SparseKernel> sks;
      int64_t off = 0;
      for (int k = 0; k < m; ++k) {
        sks.push_back(sketch(n, rp + k * (n + 1), ci + off, val + off));
        off += nnz[k];
      }
      std::vector<const SparseKernel*> kp;
      for (auto& x : sks) kp.push_back(&x);
      fill_ibp(res, ibp(kp, mp, wv, cfg, pol), q);
    } else {
      std::vector<KernelMatrix> ks;
      for (int k = 0; k < m; ++k) ks.push_back(kernel(K + k * n * n, n, 1.0, nnz_ratio[k]));
      std::vector<const KernelMatrix*> kp;
      for (auto& x : ks) kp.push_back(&x);
      fill_ibp(res, ibp(kp, mp, wv, cfg, pol), q);
    }
  });
}

int ref_spar_ibp(int32_t m, int64_t n, const double* K, const double* nnz_ratio, const double* b, const double* w,
                 double delta, int64_t max_iter, double s, uint64_t seed, int strict, double* q, ref_ibp_result* res) {
  return guard([&] {
    std::vector<DiscreteMeasure> ms;
    for (int k = 0; k < m; ++k) ms.push_back(measure(b + k * n, n));
    std::vector<const DiscreteMeasure*> mp;
    for (auto& x : ms) mp.push_back(&x);
    std::vector<KernelMatrix> ks;
    for (int k = 0; k < m; ++k) ks.push_back(kernel(K + k * n * n, n, 1.0, nnz_ratio[k]));
    std::vector<const KernelMatrix*> kp;
    for (auto& x : ks) kp.push_back(&x);
    BarycenterConfig cfg;
    cfg.delta = delta;
    cfg.max_iter = (std::size_t)max_iter;
    fill_ibp(res, spar_ibp(kp, mp, std::vector<double>(w, w + m), cfg, s, seed, strict != 0), q);
  });
}


// ---- formats (sparsify.cpp:236-263, solvers.cpp:227-242, measures.cpp:87-141, matrix.cpp) ----

int ref_save_triplet_csv(int64_t n, const int64_t* rp, const uint32_t* ci, const double* val, const char* path) {
  return guard([&] { sketch(n, rp, ci, val).save_triplet_csv(path); });
}

int ref_save_metadata_json(int64_t n, const int64_t* rp, uint64_t seed, double s, double theta, int kind,
                           const char* path) {
  return guard([&] {
    SparseKernel sk;
    sk.n = (std::size_t)n;
    sk.seed = seed;
    sk.realized_nnz = (std::size_t)rp[n];
    sk.save_metadata_json(path, s, theta, static_cast<PlanKind>(kind));
  });
}

// SolveReport::to_json into buf (sketch_nnz < 0: none)
int ref_report_json(double objective, int64_t iterations, double rr, double rc, double wall, int64_t sketch_nnz,
                    int converged, int diverged, uint64_t seed, char* buf, int64_t len) {
  return guard([&] {
    SolveReport r;
    r.objective = objective;
    r.iterations = (std::size_t)iterations;
    r.marginal_residual_row = rr;
    r.marginal_residual_col = rc;
    r.wall_time_s = wall;
    if (sketch_nnz >= 0) r.sketch_nnz = (std::size_t)sketch_nnz;
    r.converged = converged != 0;
    r.diverged = diverged != 0;
    r.seed = seed;
    std::snprintf(buf, (size_t)len, "%s", r.to_json().c_str());
  });
}

int ref_write_measure_csv(const double* w, const double* x, int64_t n, int dim, const char* path) {
  return guard([&] {
    auto m = new_measure(std::vector<double>(w, w + n), points(x, n, dim), false);
    write_measure_csv(m, path);
  });
}

int ref_read_measure_csv(const char* path, int simplex, double* w, double* x, int64_t cap, int64_t* n, int* dim) {
  return guard([&] {
    auto m = read_measure_csv(path, simplex != 0);
    *n = (int64_t)m.size();
    *dim = (int)m.support.dim;
    if (*n * *dim <= cap) {
      std::memcpy(w, m.weights.data(), sizeof(double) * m.size());
      std::memcpy(x, m.support.coords.data(), sizeof(double) * m.support.coords.size());
    }
  });
}

int ref_matrix_save(const double* a, int64_t r, int64_t c, const char* bin_path, const char* csv_path) {
  return guard([&] {
    Matrix m((std::size_t)r, (std::size_t)c);
    std::memcpy(m.data().data(), a, sizeof(double) * r * c);
    if (bin_path) m.save_binary(bin_path);
    if (csv_path) m.save_csv(csv_path);
  });
}


// ---- RMAE harness (harness.cpp:85-232) ---------------------------------------------------

static ScenarioSpec spec_of(int scenario, int64_t n, int64_t d, uint64_t seed, int has_masses, double ma, double mb,
                            int has_target, double target, double scale_param, int scale_is_sd) {
  ScenarioSpec sp;
  sp.scenario = static_cast<Scenario>(scenario);
  sp.n = (std::size_t)n;
  sp.d = (std::size_t)d;
  sp.seed = seed;
  if (has_masses) sp.masses = std::make_pair(ma, mb);
  if (has_target) sp.sparsity_target = target;
  sp.scale_param = scale_param;
  sp.scale_is_sd = scale_is_sd != 0;
  return sp;
}

// generate_scenario (+ eta_for_sparsity when a target is set)
int ref_scenario(int scenario, int64_t n, int64_t d, uint64_t seed, int has_masses, double ma, double mb,
                 int has_target, double target, double scale_param, int scale_is_sd, double* support, double* a,
                 double* b, double* eta) {
  return guard([&] {
    auto sp = spec_of(scenario, n, d, seed, has_masses, ma, mb, has_target, target, scale_param, scale_is_sd);
    ScenarioData data = generate_scenario(sp);
    std::memcpy(support, data.support.coords.data(), sizeof(double) * n * d);
    std::memcpy(a, data.a.weights.data(), sizeof(double) * n);
    std::memcpy(b, data.b.weights.data(), sizeof(double) * n);
    *eta = has_target ? eta_for_sparsity(data.support, target) : 0.0;
  });
}

int ref_rmae(int scenario, int64_t n, int64_t d, uint64_t seed, int has_masses, double ma, double mb, int has_target,
             double target, double scale_param, int scale_is_sd, int method, const double* budgets, int64_t nb,
             int64_t reps, double eps, double lambda, double delta, int64_t max_iter, double* exact, double* errors,
             int64_t* retried) {
  return guard([&] {
    auto sp = spec_of(scenario, n, d, seed, has_masses, ma, mb, has_target, target, scale_param, scale_is_sd);
    SolverConfig cfg;
    cfg.epsilon = eps;
    cfg.lambda = lambda;
    cfg.delta = delta;
    cfg.max_iter = (std::size_t)max_iter;
    RmaeReport r = rmae_experiment(sp, method ? ApproxMethod::RandSink : ApproxMethod::SparSink,
                                   std::vector<double>(budgets, budgets + nb), (std::size_t)reps, cfg);
    *exact = r.exact_objective;
    for (int64_t k = 0; k < nb; ++k) {
      retried[k] = (int64_t)r.rows[k].retried;
      for (int64_t q = 0; q < reps; ++q) errors[k * reps + q] = r.rows[k].errors[q];
    }
  });
}

}  // extern "C"
