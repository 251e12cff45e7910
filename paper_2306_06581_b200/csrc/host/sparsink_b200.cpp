// sparsink_b200.cpp -- namespace sparsink over the C ABI (libspk_b200.so).
//
// Host side above the boundary, in the reference's own language (C++), with
// the reference's names, argument meaning and exception classes
// (include/sparsink_b200.hpp lists the headers mirrored). Host work here is
// O(n) (argument checks, marshalling); every O(n^2) / O(nnz) step is a C-ABI
// call that runs on the B200. A missing device raises DeviceError -- there is
// no CPU fallback.
#include "sparsink_b200.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <sstream>

namespace sparsink {

namespace {

struct Ctx {
  spk_ctx* ctx = nullptr;
  int device = 0;
  bool deterministic = false;
  ~Ctx() {
    if (ctx) spk_ctx_destroy(ctx);
  }
};

thread_local Ctx g;

spk_ctx* ctx() {
  if (!g.ctx) {
    if (spk_ctx_create(g.device, &g.ctx) != SPK_OK) {
      g.ctx = nullptr;
      throw DeviceError("sparsink_b200: no usable CUDA device " + std::to_string(g.device));
    }
    spk_ctx_set_option(g.ctx, SPK_OPT_DETERMINISTIC, g.deterministic ? 1 : 0);
  }
  return g.ctx;
}

std::string strip(const std::string& msg, const char* cls) {
  const std::string p = std::string(cls) + ": ";
  return msg.compare(0, p.size(), p) == 0 ? msg.substr(p.size()) : msg;
}

// Rethrow the C-ABI failure as the reference's exception class.
[[noreturn]] void rethrow(spk_ctx* c) {
  int cat = 0, kind = 0;
  char buf[1024];
  spk_last_error(c, &cat, &kind, buf, sizeof buf);
  const std::string m = buf;
#define K(code, Cls) \
  case code: throw Cls(strip(m, #Cls));
  switch (kind) {
    K(SPK_E_NEGATIVE_WEIGHT, NegativeWeight)
    K(SPK_E_LENGTH_MISMATCH, LengthMismatch)
    K(SPK_E_NOT_NORMALIZED, NotNormalized)
    K(SPK_E_ALL_BLACK, AllBlack)
    K(SPK_E_EMPTY_OUTPUT, EmptyOutput)
    K(SPK_E_DIMENSION_MISMATCH, DimensionMismatch)
    K(SPK_E_NON_POSITIVE_ETA, NonPositiveEta)
    K(SPK_E_NON_POSITIVE_EPSILON, NonPositiveEpsilon)
    K(SPK_E_DEGENERATE_SUPPORT, DegenerateSupport)
    K(SPK_E_ALL_ZERO_KERNEL, AllZeroKernel)
    K(SPK_E_THETA_OUT_OF_RANGE, ThetaOutOfRange)
    K(SPK_E_BUDGET_TOO_LARGE, BudgetTooLarge)
    K(SPK_E_EMPTY_WINDOW, EmptyWindow)
    K(SPK_E_INFINITE_COST_ON_SUPPORT, InfiniteCostOnSupport)
    K(SPK_E_IO_ERROR, IoError)
    K(SPK_E_ZERO_DENOMINATOR, ZeroDenominator)
    K(SPK_E_BASELINE_FAILED, BaselineFailed)
    K(SPK_E_DEGENERATE_SKETCH_ERROR, DegenerateSketchError)
    case SPK_E_DEVICE: throw DeviceError(m);
    default: throw Error(static_cast<ErrorCategory>(cat == 0 ? 4 : cat), m);
  }
#undef K
}

void check(int rc) {
  if (rc != SPK_OK) rethrow(ctx());
}

// Reference exception class name of a spk_error_kind.
std::string error_class_name(int kind) {
  static const char* const names[] = {"",
                                      "Error",
                                      "NegativeWeight",
                                      "LengthMismatch",
                                      "NotNormalized",
                                      "AllBlack",
                                      "EmptyOutput",
                                      "DimensionMismatch",
                                      "NonPositiveEta",
                                      "NonPositiveEpsilon",
                                      "DegenerateSupport",
                                      "AllZeroKernel",
                                      "ThetaOutOfRange",
                                      "BudgetTooLarge",
                                      "EmptyWindow",
                                      "InfiniteCostOnSupport",
                                      "IoError",
                                      "ZeroDenominator",
                                      "BaselineFailed",
                                      "DegenerateSketchError",
                                      "DeviceError"};
  return kind >= 0 && kind <= 20 ? names[kind] : "Error";
}

int kind_of(CostKind k) {
  return k == CostKind::SqEuclidean ? SPK_COST_SQEUCLID : k == CostKind::Euclidean ? SPK_COST_EUCLID : SPK_COST_WFR;
}

spk_kernel_desc dense_desc(const KernelMatrix& K, const CostMatrix* C) {
  spk_kernel_desc d{};
  d.n = static_cast<int64_t>(K.size());
  d.K = K.entries.data().data();
  d.nnz_ratio = K.nnz_ratio;
  d.C = C ? C->entries.data().data() : nullptr;
  d.kernel_epsilon = K.epsilon > 0.0 ? K.epsilon : 0.0;
  return d;
}

spk_kernel_desc coord_desc(const PointList& x, const PointList& y, const CostSpec& cs, double eps) {
  if (x.dim != y.dim || x.dim == 0) throw DimensionMismatch("point lists must share a positive dimension");
  if (x.size() != y.size()) throw LengthMismatch("coordinate overloads need n source and n target points");
  spk_kernel_desc d{};
  d.n = static_cast<int64_t>(x.size());
  d.x = x.coords.data();
  d.y = y.coords.data();
  d.dim = static_cast<int32_t>(x.dim);
  d.cost_kind = kind_of(cs.kind);
  d.eta = cs.eta;
  d.cost_scale = cs.scale;
  d.kernel_epsilon = eps;
  return d;
}

spk_solver_cfg c_cfg(const SolverConfig& cfg, EmptyPolicy policy) {
  spk_solver_cfg c{};
  c.epsilon = cfg.epsilon;
  c.lambda = cfg.lambda;
  c.delta = cfg.delta;
  c.max_iter = static_cast<int64_t>(cfg.max_iter);
  c.stabilize = cfg.stabilize ? 1 : 0;
  c.empty_policy = policy == EmptyPolicy::Mask ? SPK_POLICY_MASK : SPK_POLICY_ERROR;
  return c;
}

spk_sketch_opts c_opts(const SparSinkOptions& o) {
  spk_sketch_opts s{};
  s.theta = o.theta;
  s.probs = o.probs == SketchProbs::Uniform ? SPK_PROBS_UNIFORM : SPK_PROBS_IMPORTANCE;
  s.strict = o.strict ? 1 : 0;
  s.value_type = o.values == ValuePrecision::F32 ? SPK_VALUES_F32 : SPK_VALUES_F64;
  return s;
}

void check_sizes(std::size_t n, const DiscreteMeasure& a, const DiscreteMeasure& b) {
  if (a.size() != n || b.size() != n) throw LengthMismatch("measure size does not match kernel dimension");
}

SolveResult make_result(std::size_t n, const spk_report& r, std::vector<double> u, std::vector<double> v,
                        std::vector<double> lu, std::vector<double> lv) {
  SolveResult res;
  res.plan.u = std::move(u);
  res.plan.v = std::move(v);
  res.plan.log_domain = r.log_domain != 0;
  if (res.plan.log_domain) {
    res.plan.log_u = std::move(lu);
    res.plan.log_v = std::move(lv);
  }
  res.plan.converged = r.converged != 0;
  res.plan.iterations = static_cast<std::size_t>(r.iterations);
  res.plan.masked_rows = static_cast<std::size_t>(r.masked_rows);
  res.plan.masked_cols = static_cast<std::size_t>(r.masked_cols);
  res.report.iterations = static_cast<std::size_t>(r.iterations);
  res.report.marginal_residual_row = r.residual_row;
  res.report.marginal_residual_col = r.residual_col;
  res.report.wall_time_s = r.wall_time_s;
  res.report.converged = r.converged != 0;
  res.report.diverged = r.diverged != 0;
  res.report.kernel_mean = r.kernel_mean;
  (void)n;
  return res;
}

struct DeviceSketch {  // a host SparseKernel uploaded for one call
  spk_sketch* sk = nullptr;
  explicit DeviceSketch(const SparseKernel& M) {
    std::vector<int64_t> rp(M.row_ptr.begin(), M.row_ptr.end());
    check(spk_sketch_from_csr(ctx(), static_cast<int64_t>(M.n), rp.data(), M.col_idx.data(), M.values.data(),
                              SPK_VALUES_F64, &sk));
  }
  ~DeviceSketch() { spk_sketch_free(sk); }
};

SolveResult dense_solve(const KernelMatrix& K, const DiscreteMeasure& a, const DiscreteMeasure& b,
                        const SolverConfig& cfg, EmptyPolicy policy, bool uot) {
  const std::size_t n = K.size();
  check_sizes(n, a, b);
  spk_kernel_desc d = dense_desc(K, nullptr);
  spk_solver_cfg c = c_cfg(cfg, policy);
  std::vector<double> u(n), v(n), lu(n), lv(n);
  spk_report r;
  check(spk_sinkhorn(ctx(), &d, a.weights.data(), b.weights.data(), &c, uot ? 1 : 0, u.data(), v.data(), lu.data(),
                     lv.data(), &r));
  SolveResult res = make_result(n, r, std::move(u), std::move(v), std::move(lu), std::move(lv));
  res.plan.dense_kernel = &K;
  return res;  // objective stays NaN: sinkhorn_* callers evaluate it (reference semantics)
}

SolveResult sparse_solve(const SparseKernel& K, const DiscreteMeasure& a, const DiscreteMeasure& b,
                         const SolverConfig& cfg, EmptyPolicy policy, bool uot) {
  const std::size_t n = K.n;
  check_sizes(n, a, b);
  DeviceSketch ds(K);
  spk_solver_cfg c = c_cfg(cfg, policy);
  std::vector<double> u(n), v(n), lu(n), lv(n);
  spk_report r;
  check(spk_sketch_solve(ctx(), ds.sk, a.weights.data(), b.weights.data(), &c, uot ? 1 : 0, u.data(), v.data(),
                         lu.data(), lv.data(), &r));
  SolveResult res = make_result(n, r, std::move(u), std::move(v), std::move(lu), std::move(lv));
  res.plan.sparse_kernel = &K;
  return res;
}

SolveResult spar_sink(const spk_kernel_desc& d, const DiscreteMeasure& a, const DiscreteMeasure& b,
                      const SolverConfig& cfg, double s, std::uint64_t seed, const SparSinkOptions& opts, bool uot) {
  const std::size_t n = static_cast<std::size_t>(d.n);
  check_sizes(n, a, b);
  spk_solver_cfg c = c_cfg(cfg, EmptyPolicy::Mask);
  spk_sketch_opts o = c_opts(opts);
  std::vector<double> u(n), v(n), lu(n), lv(n);
  spk_report r;
  if (!opts.devices.empty() && d.x) {  // rows / columns sharded over the listed GPUs of this process
    const int rc = spk_spar_sink_multi(opts.devices.data(), static_cast<int>(opts.devices.size()), &d,
                                       a.weights.data(), b.weights.data(), &c, s, seed, &o, uot ? 1 : 0, u.data(),
                                       v.data(), lu.data(), lv.data(), &r);
    if (rc != SPK_OK) rethrow(nullptr);
  } else {
    check(spk_spar_sink(ctx(), &d, a.weights.data(), b.weights.data(), &c, s, seed, &o, uot ? 1 : 0, u.data(),
                        v.data(), lu.data(), lv.data(), &r));
  }
  SolveResult res = make_result(n, r, std::move(u), std::move(v), std::move(lu), std::move(lv));
  res.report.objective = r.objective;
  res.report.sketch_nnz = static_cast<std::size_t>(r.sketch_nnz);
  res.report.seed = seed;
  res.report.wall_time_s = r.wall_time_s;
  return res;  // plan.sparse_kernel stays null: the sketch died with the call (solvers.cpp:356)
}

// Readout of a plan through the device (marginals, objective, residuals).
struct Readout {
  std::vector<double> row, col;
  double objective = std::numeric_limits<double>::quiet_NaN();
  double rr = 0.0, rc = 0.0;
};

Readout plan_readout(const TransportPlan& T, const CostMatrix* C, const DiscreteMeasure* a, const DiscreteMeasure* b,
                     bool uot, double lambda, double eps, bool want_obj) {
  const std::size_t n = T.size();
  Readout out;
  out.row.assign(n, 0.0);
  out.col.assign(n, 0.0);
  if (!T.dense_kernel && !T.sparse_kernel) return out;  // reference: no kernel -> no entries
  spk_kernel_desc d{};
  std::vector<int64_t> rp;
  const int64_t* rpp = nullptr;
  const uint32_t* ci = nullptr;
  const double* vv = nullptr;
  if (T.dense_kernel) {
    d = dense_desc(*T.dense_kernel, C);
  } else {
    rp.assign(T.sparse_kernel->row_ptr.begin(), T.sparse_kernel->row_ptr.end());
    rpp = rp.data();
    ci = T.sparse_kernel->col_idx.data();
    vv = T.sparse_kernel->values.data();
    d.n = static_cast<int64_t>(n);
    d.C = C ? C->entries.data().data() : nullptr;  // cost-only form
  }
  const bool have_desc = T.dense_kernel || C;
  check(spk_plan_readout(ctx(), have_desc ? &d : nullptr, static_cast<int64_t>(n), rpp, ci, vv, T.u.data(), T.v.data(),
                         T.log_domain ? T.log_u.data() : nullptr, T.log_domain ? T.log_v.data() : nullptr,
                         T.log_domain ? 1 : 0, a ? a->weights.data() : nullptr, b ? b->weights.data() : nullptr,
                         uot ? 1 : 0, lambda, eps, out.row.data(), out.col.data(), want_obj ? &out.objective : nullptr,
                         &out.rr, &out.rc));
  return out;
}

}  // namespace

void set_device(int device) {
  if (g.ctx) {
    spk_ctx_destroy(g.ctx);
    g.ctx = nullptr;
  }
  g.device = device;
}

void set_deterministic(bool on) {
  g.deterministic = on;
  if (g.ctx) spk_ctx_set_option(g.ctx, SPK_OPT_DETERMINISTIC, on ? 1 : 0);
}

// measures.cpp:12-34
DiscreteMeasure new_measure(std::vector<double> weights, PointList support, bool require_simplex) {
  if (weights.empty()) throw LengthMismatch("measure must have atoms");
  if (support.dim == 0 || support.coords.size() != weights.size() * support.dim)
    throw LengthMismatch("support length must equal weights length");
  double total = 0.0;
  bool any_positive = false;
  for (double w : weights) {
    if (w < 0.0 || !std::isfinite(w)) throw NegativeWeight("weight " + std::to_string(w));
    any_positive = any_positive || w > 0.0;
    total += w;
  }
  if (!any_positive) throw NegativeWeight("all weights are zero");
  if (require_simplex && std::abs(total - 1.0) > 1e-8) throw NotNormalized("weights sum to " + std::to_string(total));
  DiscreteMeasure m;
  m.weights = std::move(weights);
  m.support = std::move(support);
  m.total_mass = total;
  return m;
}

namespace {
CostMatrix pairwise(const PointList& x, const PointList& y, CostKind kind, double eta) {
  if (x.dim != y.dim || x.dim == 0) throw DimensionMismatch("point lists must share a positive dimension");
  const std::size_t nx = x.size(), ny = y.size(), n = std::max(nx, ny);
  // the C ABI takes n x and n y points: pad the shorter list (padded pairs are not queried)
  std::vector<double> xp(x.coords), yp(y.coords);
  xp.resize(n * x.dim, 0.0);
  yp.resize(n * y.dim, 0.0);
  spk_kernel_desc d{};
  d.n = static_cast<int64_t>(n);
  d.x = xp.data();
  d.y = yp.data();
  d.dim = static_cast<int32_t>(x.dim);
  d.cost_kind = kind_of(kind);
  d.eta = eta;
  d.cost_scale = 1.0;
  d.kernel_epsilon = 1.0;
  std::vector<int64_t> qi(nx * ny), qj(nx * ny);
  for (std::size_t i = 0; i < nx; ++i)
    for (std::size_t j = 0; j < ny; ++j) {
      qi[i * ny + j] = static_cast<int64_t>(i);
      qj[i * ny + j] = static_cast<int64_t>(j);
    }
  CostMatrix c;
  c.kind = kind;
  c.eta = eta;
  c.entries = Matrix(nx, ny);
  check(spk_cost_kernel(ctx(), &d, static_cast<int64_t>(nx * ny), qi.data(), qj.data(), c.entries.data().data(),
                        nullptr, nullptr));
  double c0 = 0.0;
  for (double v : c.entries.data())
    if (std::isfinite(v) && v > c0) c0 = v;  // geometry.cpp:61
  c.c0 = c0;
  return c;
}
}  // namespace

CostMatrix sq_euclidean_cost(const PointList& x, const PointList& y) {
  return pairwise(x, y, CostKind::SqEuclidean, 0.0);
}
CostMatrix euclidean_cost(const PointList& x, const PointList& y) { return pairwise(x, y, CostKind::Euclidean, 0.0); }
CostMatrix wfr_cost(const PointList& x, const PointList& y, double eta) {
  if (!(eta > 0.0)) throw NonPositiveEta("eta = " + std::to_string(eta));
  return pairwise(x, y, CostKind::WFR, eta);
}

KernelMatrix kernel_from_cost(const CostMatrix& cost, double epsilon) {
  if (!(epsilon > 0.0)) throw NonPositiveEpsilon("epsilon = " + std::to_string(epsilon));
  KernelMatrix K;
  K.epsilon = epsilon;
  K.entries = Matrix(cost.entries.rows(), cost.entries.cols());
  int64_t nnz = 0;
  const int64_t m = static_cast<int64_t>(cost.entries.data().size());
  check(spk_kernel_from_cost(ctx(), cost.entries.data().data(), m, epsilon, K.entries.data().data(), &nnz));
  K.nnz_ratio = static_cast<double>(nnz) / static_cast<double>(m);
  return K;
}

// ---- plans & sketches ---------------------------------------------------------------------
struct PlanAccess {
  static const std::vector<double>& a(const SamplingPlan& p) { return p.a_; }
  static const std::vector<double>& b(const SamplingPlan& p) { return p.b_; }
  static double lambda(const SamplingPlan& p) { return p.lambda_; }
  static double epsilon(const SamplingPlan& p) { return p.epsilon_; }
  static int kind(PlanKind k) {
    switch (k) {
      case PlanKind::OT: return SPK_PLAN_OT;
      case PlanKind::UOT: return SPK_PLAN_UOT;
      case PlanKind::Barycenter: return SPK_PLAN_BARYCENTER;
      default: return SPK_PLAN_UNIFORM;
    }
  }
};

namespace {
void check_plan_sizes(const DiscreteMeasure& a, const DiscreteMeasure& b, const KernelMatrix& K) {
  if (a.size() != K.size() || b.size() != K.size()) throw LengthMismatch("measures must match kernel dimension");
  if (std::llround(K.nnz_ratio * static_cast<double>(K.size()) * static_cast<double>(K.size())) == 0)
    throw AllZeroKernel("kernel has no support");
}
}  // namespace

SamplingPlan ot_probabilities(const DiscreteMeasure& a, const DiscreteMeasure& b, const KernelMatrix& K) {
  check_plan_sizes(a, b, K);
  SamplingPlan p;
  p.kind_ = PlanKind::OT;
  p.kernel_ = &K;
  p.a_ = a.weights;
  p.b_ = b.weights;
  p.epsilon_ = K.epsilon > 0 ? K.epsilon : 1.0;
  p.factorized_storage();  // surfaces AllZeroKernel("zero-mass measure") eagerly
  return p;
}

SamplingPlan uot_probabilities(const DiscreteMeasure& a, const DiscreteMeasure& b, const KernelMatrix& K,
                               double lambda, double epsilon) {
  if (!(lambda > 0.0)) throw Error(ErrorCategory::Input, "lambda must be > 0");
  if (!(epsilon > 0.0)) throw NonPositiveEpsilon("uot_probabilities");
  check_plan_sizes(a, b, K);
  SamplingPlan p;
  p.kind_ = PlanKind::UOT;
  p.kernel_ = &K;
  p.a_ = a.weights;
  p.b_ = b.weights;
  p.lambda_ = lambda;
  p.epsilon_ = epsilon;
  p.factorized_storage();
  return p;
}

SamplingPlan uniform_probabilities(const KernelMatrix& K) {
  if (std::llround(K.nnz_ratio * static_cast<double>(K.size()) * static_cast<double>(K.size())) == 0)
    throw AllZeroKernel("kernel has no support");
  SamplingPlan p;
  p.kind_ = PlanKind::Uniform;
  p.kernel_ = &K;
  p.a_.assign(K.size(), 1.0);
  p.b_.assign(K.size(), 1.0);
  return p;
}

SamplingPlan barycenter_probabilities(const DiscreteMeasure& b_k, const KernelMatrix& K_k) {
  check_plan_sizes(b_k, b_k, K_k);
  SamplingPlan p;
  p.kind_ = PlanKind::Barycenter;
  p.kernel_ = &K_k;
  p.a_.assign(K_k.size(), 1.0);  // unused by the column-constant plan
  p.b_ = b_k.weights;
  p.epsilon_ = K_k.epsilon > 0 ? K_k.epsilon : 1.0;
  p.factorized_storage();  // surfaces AllZeroKernel("zero-mass measure") eagerly
  return p;
}

double eta_for_sparsity(const PointList& x, double target_nnz_ratio) {
  if (!(target_nnz_ratio > 0.0 && target_nnz_ratio <= 1.0))
    throw ThetaOutOfRange("target nnz ratio must lie in (0,1]");
  const std::size_t n = x.size();
  if (n < 2) throw DegenerateSupport("need at least two points");
  // all n^2 distances (the pairwise cost on the device, Euclidean form)
  CostMatrix d = euclidean_cost(x, x);
  std::vector<double>& v = d.entries.data();
  const double dmax = *std::max_element(v.begin(), v.end());
  if (dmax == 0.0) {
    if (target_nnz_ratio < 1.0) throw DegenerateSupport("all points identical");
    return 1.0;
  }
  constexpr double kPi = 3.14159265358979323846;
  if (target_nnz_ratio >= 1.0) return dmax / kPi * 1.0001 + 1e-12;
  const std::size_t keep = std::max<std::size_t>(
      1, static_cast<std::size_t>(std::llround(target_nnz_ratio * static_cast<double>(n) * static_cast<double>(n))));
  // the kept quantile and the next one: two order statistics, no full sort
  std::nth_element(v.begin(), v.begin() + (keep - 1), v.end());
  const double q_in = v[keep - 1];
  const double q_out = keep < v.size() ? *std::min_element(v.begin() + keep, v.end()) : q_in * 1.0001;
  return (q_in == q_out ? q_in * (1.0 + 1e-9) : 0.5 * (q_in + q_out)) / kPi;
}

SamplingPlan shrink_with_uniform(const SamplingPlan& plan, double theta) {
  if (!(theta >= 0.0 && theta < 1.0)) throw ThetaOutOfRange("theta = " + std::to_string(theta));
  SamplingPlan out = plan;
  out.theta_ = theta;
  return out;
}

bool SamplingPlan::factorized_storage() const {
  spk_kernel_desc d = dense_desc(*kernel_, nullptr);
  int32_t fac = 0;
  check(spk_plan_probs(ctx(), &d, a_.data(), b_.data(), PlanAccess::kind(kind_), lambda_, epsilon_, theta_, 0, nullptr,
                       nullptr, nullptr, &fac));
  return fac != 0;
}

double SamplingPlan::prob(std::size_t i, std::size_t j) const {
  spk_kernel_desc d = dense_desc(*kernel_, nullptr);
  const int64_t qi = static_cast<int64_t>(i), qj = static_cast<int64_t>(j);
  double p = 0.0;
  int32_t fac = 0;
  check(spk_plan_probs(ctx(), &d, a_.data(), b_.data(), PlanAccess::kind(kind_), lambda_, epsilon_, theta_, 1, &qi,
                       &qj, &p, &fac));
  return p;
}

SparseKernel poisson_sparsify(const KernelMatrix& K, const SamplingPlan& plan, double s, std::uint64_t seed) {
  if (plan.size() != K.size()) throw LengthMismatch("plan dimension != kernel");
  spk_kernel_desc d = dense_desc(K, nullptr);
  spk_sketch_opts o{};
  o.theta = plan.theta();
  o.value_type = SPK_VALUES_F64;
  spk_sketch* sk = nullptr;
  check(spk_sketch_build(ctx(), &d, PlanAccess::a(plan).data(), PlanAccess::b(plan).data(),
                         PlanAccess::kind(plan.kind()), PlanAccess::lambda(plan), PlanAccess::epsilon(plan), s, seed,
                         &o, &sk));
  int64_t n = 0, nnz = 0;
  spk_sketch_info(sk, &n, &nnz, nullptr, nullptr, nullptr);
  std::vector<int64_t> rp(n + 1);
  SparseKernel out;
  out.n = static_cast<std::size_t>(n);
  out.seed = seed;
  out.epsilon = K.epsilon;
  out.col_idx.resize(nnz);
  out.values.resize(nnz);
  const int rc = spk_sketch_copy_csr(sk, rp.data(), out.col_idx.data(), out.values.data());
  spk_sketch_free(sk);
  check(rc);
  out.row_ptr.assign(rp.begin(), rp.end());
  out.realized_nnz = static_cast<std::size_t>(nnz);
  return out;
}

Matrix SparseKernel::to_dense() const {
  Matrix m(n, n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) m(i, col_idx[p]) = values[p];
  return m;
}

namespace {
std::vector<double> product(const SparseKernel& M, const std::vector<double>& x, int transpose) {
  if (x.size() != M.n) throw LengthMismatch(transpose ? "spmv_t vector length" : "spmv vector length");
  DeviceSketch ds(M);
  std::vector<double> y(M.n);
  check(spk_sketch_spmv(ds.sk, x.data(), y.data(), transpose));
  return y;
}
}  // namespace

std::vector<double> spmv(const SparseKernel& M, const std::vector<double>& v) { return product(M, v, 0); }
std::vector<double> spmv_t(const SparseKernel& M, const std::vector<double>& u) { return product(M, u, 1); }

// ---- solvers ----------------------------------------------------------------------------
template <>
SolveResult sinkhorn_ot<KernelMatrix>(const KernelMatrix& K, const DiscreteMeasure& a, const DiscreteMeasure& b,
                                      const SolverConfig& cfg, EmptyPolicy p) {
  return dense_solve(K, a, b, cfg, p, false);
}
template <>
SolveResult sinkhorn_uot<KernelMatrix>(const KernelMatrix& K, const DiscreteMeasure& a, const DiscreteMeasure& b,
                                       const SolverConfig& cfg, EmptyPolicy p) {
  return dense_solve(K, a, b, cfg, p, true);
}
template <>
SolveResult sinkhorn_ot<SparseKernel>(const SparseKernel& K, const DiscreteMeasure& a, const DiscreteMeasure& b,
                                      const SolverConfig& cfg, EmptyPolicy p) {
  return sparse_solve(K, a, b, cfg, p, false);
}
template <>
SolveResult sinkhorn_uot<SparseKernel>(const SparseKernel& K, const DiscreteMeasure& a, const DiscreteMeasure& b,
                                       const SolverConfig& cfg, EmptyPolicy p) {
  return sparse_solve(K, a, b, cfg, p, true);
}

SolveResult spar_sink_ot(const KernelMatrix& K, const CostMatrix& C, const DiscreteMeasure& a,
                         const DiscreteMeasure& b, const SolverConfig& cfg, double s, std::uint64_t seed,
                         const SparSinkOptions& opts) {
  return spar_sink(dense_desc(K, &C), a, b, cfg, s, seed, opts, false);
}

SolveResult spar_sink_uot(const KernelMatrix& K, const CostMatrix& C, const DiscreteMeasure& a,
                          const DiscreteMeasure& b, const SolverConfig& cfg, double s, std::uint64_t seed,
                          const SparSinkOptions& opts) {
  return spar_sink(dense_desc(K, &C), a, b, cfg, s, seed, opts, true);
}

SolveResult spar_sink_ot(const PointList& x, const PointList& y, const CostSpec& cost, const DiscreteMeasure& a,
                         const DiscreteMeasure& b, const SolverConfig& cfg, double s, std::uint64_t seed,
                         const SparSinkOptions& opts) {
  return spar_sink(coord_desc(x, y, cost, cfg.epsilon), a, b, cfg, s, seed, opts, false);
}

SolveResult spar_sink_uot(const PointList& x, const PointList& y, const CostSpec& cost, const DiscreteMeasure& a,
                          const DiscreteMeasure& b, const SolverConfig& cfg, double s, std::uint64_t seed,
                          const SparSinkOptions& opts) {
  return spar_sink(coord_desc(x, y, cost, cfg.epsilon), a, b, cfg, s, seed, opts, true);
}

std::vector<PairSolve> spar_sink_uot_pairs(const PointList& support, const CostSpec& cost,
                                           const std::vector<DiscreteMeasure>& measures,
                                           const std::vector<std::pair<std::size_t, std::size_t>>& pairs,
                                           const SolverConfig& cfg, double s, const std::vector<std::uint64_t>& seeds,
                                           const SparSinkOptions& opts) {
  if (seeds.size() != pairs.size()) throw LengthMismatch("one seed per pair");
  const spk_kernel_desc d = coord_desc(support, support, cost, cfg.epsilon);
  const std::size_t n = static_cast<std::size_t>(d.n);
  for (const auto& pr : pairs) {
    if (pr.first >= measures.size() || pr.second >= measures.size()) throw LengthMismatch("pair index out of range");
    check_sizes(n, measures[pr.first], measures[pr.second]);
  }
  const spk_solver_cfg c = c_cfg(cfg, opts.strict ? EmptyPolicy::Error : EmptyPolicy::Mask);
  const spk_sketch_opts o = c_opts(opts);
  std::vector<PairSolve> out(pairs.size());
  constexpr std::size_t kChunk = 512;  // sketches resident at once
  for (std::size_t c0 = 0; c0 < pairs.size(); c0 += kChunk) {
    const std::size_t m = std::min(kChunk, pairs.size() - c0);
    std::vector<double> A(m * n), B(m * n);
    for (std::size_t q = 0; q < m; ++q) {
      std::copy(measures[pairs[c0 + q].first].weights.begin(), measures[pairs[c0 + q].first].weights.end(),
                A.begin() + q * n);
      std::copy(measures[pairs[c0 + q].second].weights.begin(), measures[pairs[c0 + q].second].weights.end(),
                B.begin() + q * n);
    }
    std::vector<spk_sketch*> sks(m, nullptr);
    check(spk_sketch_build_batch(ctx(), &d, static_cast<int>(m), A.data(), B.data(), SPK_PLAN_UOT, cfg.lambda,
                                 cfg.epsilon, s, seeds.data() + c0, &o, sks.data()));
    struct Free {  // the chunk's sketches die with the chunk, whatever happens
      std::vector<spk_sketch*>& v;
      ~Free() {
        for (spk_sketch* p : v) spk_sketch_free(p);
      }
    } free_all{sks};
    std::vector<spk_report> reps(m);
    std::vector<int32_t> err(m, 0);
    check(spk_sketch_solve_batch(ctx(), sks.data(), static_cast<int>(m), &c, 1, reps.data(), err.data()));
    for (std::size_t q = 0; q < m; ++q) {
      PairSolve& ps = out[c0 + q];
      if (err[q]) {
        ps.failed = true;
        ps.error = error_class_name(err[q]);
        ps.result.report.objective = std::numeric_limits<double>::quiet_NaN();
        ps.result.report.seed = seeds[c0 + q];
        continue;
      }
      std::vector<double> u(n), v(n), lu(n), lv(n);
      check(spk_sketch_scalings(sks[q], u.data(), v.data(), lu.data(), lv.data()));
      double obj = std::numeric_limits<double>::quiet_NaN();
      spk_report rr = reps[q];
      if (spk_sketch_readout(ctx(), sks[q], &d, 1, cfg.lambda, cfg.epsilon, nullptr, nullptr, &obj, &rr) != SPK_OK) {
        int cat = 0, kind = 0;
        spk_last_error(ctx(), &cat, &kind, nullptr, 0);
        if (kind == SPK_E_DEVICE) rethrow(ctx());
        ps.failed = true;
        ps.error = error_class_name(kind);
        ps.result.report.objective = std::numeric_limits<double>::quiet_NaN();
        ps.result.report.seed = seeds[c0 + q];
        continue;
      }
      ps.result = make_result(n, reps[q], std::move(u), std::move(v), std::move(lu), std::move(lv));
      ps.result.report.objective = obj;
      ps.result.report.sketch_nnz = static_cast<std::size_t>(reps[q].sketch_nnz);
      ps.result.report.seed = seeds[c0 + q];
    }
  }
  return out;
}

namespace {
SolveResult otf_solve(const PointList& x, const PointList& y, const CostSpec& cost, const DiscreteMeasure& a,
                      const DiscreteMeasure& b, const SolverConfig& cfg, EmptyPolicy p, bool uot) {
  spk_kernel_desc d = coord_desc(x, y, cost, cfg.epsilon);
  const std::size_t n = static_cast<std::size_t>(d.n);
  check_sizes(n, a, b);
  spk_solver_cfg c = c_cfg(cfg, p);
  std::vector<double> u(n), v(n), lu(n), lv(n);
  spk_report r;
  check(spk_sinkhorn(ctx(), &d, a.weights.data(), b.weights.data(), &c, uot ? 1 : 0, u.data(), v.data(), lu.data(),
                     lv.data(), &r));
  SolveResult res = make_result(n, r, std::move(u), std::move(v), std::move(lu), std::move(lv));
  res.report.objective = r.objective;  // the on-the-fly solve reads the objective out on the device
  return res;
}
}  // namespace

SolveResult sinkhorn_ot(const PointList& x, const PointList& y, const CostSpec& cost, const DiscreteMeasure& a,
                        const DiscreteMeasure& b, const SolverConfig& cfg, EmptyPolicy p) {
  constexpr double kSimplexTol = 1e-8;
  if (std::abs(a.total_mass - 1.0) > kSimplexTol || std::abs(b.total_mass - 1.0) > kSimplexTol)
    throw NotNormalized("sinkhorn_ot requires simplex inputs");
  return otf_solve(x, y, cost, a, b, cfg, p, false);
}

SolveResult sinkhorn_uot(const PointList& x, const PointList& y, const CostSpec& cost, const DiscreteMeasure& a,
                         const DiscreteMeasure& b, const SolverConfig& cfg, EmptyPolicy p) {
  return otf_solve(x, y, cost, a, b, cfg, p, true);
}

// ---- plan readout -------------------------------------------------------------------------
double TransportPlan::entry(std::size_t i, std::size_t j) const {
  double kij = 0.0;
  if (dense_kernel) {
    kij = dense_kernel->entries(i, j);
  } else if (sparse_kernel) {
    for (std::size_t p = sparse_kernel->row_ptr[i]; p < sparse_kernel->row_ptr[i + 1]; ++p)
      if (sparse_kernel->col_idx[p] == j) {
        kij = sparse_kernel->values[p];
        break;
      }
  }
  if (kij == 0.0) return 0.0;
  if (log_domain) {
    if (log_u[i] == -std::numeric_limits<double>::infinity() || log_v[j] == -std::numeric_limits<double>::infinity())
      return 0.0;
    return std::exp(log_u[i] + std::log(kij) + log_v[j]);
  }
  return u[i] * kij * v[j];
}

std::vector<double> TransportPlan::row_marginal() const {
  return plan_readout(*this, nullptr, nullptr, nullptr, false, 0.0, 1.0, false).row;
}

std::vector<double> TransportPlan::col_marginal() const {
  return plan_readout(*this, nullptr, nullptr, nullptr, false, 0.0, 1.0, false).col;
}

double ot_objective(const TransportPlan& T, const CostMatrix& C, double epsilon) {
  return plan_readout(T, &C, nullptr, nullptr, false, 0.0, epsilon, true).objective;
}

double uot_objective(const TransportPlan& T, const CostMatrix& C, const DiscreteMeasure& a, const DiscreteMeasure& b,
                     double lambda, double epsilon) {
  return plan_readout(T, &C, &a, &b, true, lambda, epsilon, true).objective;
}

std::pair<double, double> marginal_residuals(const TransportPlan& T, const DiscreteMeasure& a,
                                             const DiscreteMeasure& b) {
  if (T.size() != a.size() || T.size() != b.size()) throw LengthMismatch("marginal_residuals");
  Readout r = plan_readout(T, nullptr, &a, &b, false, 0.0, 1.0, false);
  return {r.rr, r.rc};
}

// solvers.cpp:246-260 (O(n) host arithmetic on two vectors)
double kl_divergence(const std::vector<double>& x, const std::vector<double>& y) {
  if (x.size() != y.size()) throw LengthMismatch("kl_divergence");
  double acc = 0.0;
  for (std::size_t i = 0; i < x.size(); ++i) {
    if (x[i] > 0.0) {
      if (y[i] <= 0.0) throw Error(ErrorCategory::Input, "KL undefined: mass off support");
      acc += x[i] * std::log(x[i] / y[i]) - x[i] + y[i];
    } else {
      acc += y[i];
    }
  }
  return acc;
}

std::string SolveReport::to_json() const {
  std::ostringstream o;
  o.precision(17);
  o << "{\n  \"objective\": " << objective << ",\n  \"iterations\": " << iterations
    << ",\n  \"residual_row\": " << marginal_residual_row << ",\n  \"residual_col\": " << marginal_residual_col
    << ",\n  \"wall_time_s\": " << wall_time_s << ",\n  \"sketch_nnz\": ";
  if (sketch_nnz) o << *sketch_nnz;
  else o << "null";
  o << ",\n  \"converged\": " << (converged ? "true" : "false") << ",\n  \"diverged\": "
    << (diverged ? "true" : "false") << ",\n  \"seed\": " << seed << "\n}";
  return o.str();
}

}  // namespace sparsink
