// C++ drop-in check: the reference's own unit-test scenarios
// (proj/tests/test_solvers.cpp, test_sparsify.cpp, test_geometry.cpp),
// restated against namespace sparsink from include/sparsink_b200.hpp, i.e.
// the same calls a reference user makes -- now served by the B200.
// Run by tests/test_cpp_dropin.py (GPU box). Exit status = #failures.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "sparsink_b200.hpp"

using namespace sparsink;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    if (cond) ++g_pass;                                                     \
    else {                                                                  \
      ++g_fail;                                                             \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                       \
  } while (0)
#define CHECK_CLOSE(a, b, rel) CHECK(std::abs((a) - (b)) <= (rel) * std::abs(b))
#define CHECK_THROWS_AS(expr, T)                 \
  do {                                           \
    bool caught_ = false;                        \
    try {                                        \
      (void)(expr);                              \
    } catch (const T&) {                         \
      caught_ = true;                            \
    } catch (...) {                              \
    }                                            \
    CHECK(caught_ && #T);                        \
  } while (0)

static void run(const char* name, const std::function<void()>& f) {
  const int before = g_fail;
  try {
    f();
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("  FAIL exception: %s\n", e.what());
  }
  std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

static PointList pts1d(std::initializer_list<double> xs) {
  PointList p;
  p.dim = 1;
  p.coords = xs;
  return p;
}

// splitmix64 counter stream, as the reference's CounterRng (rng.hpp:10-40)
static double draw(std::uint64_t seed, std::uint64_t stream, std::uint64_t t) {
  auto sm = [](std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  };
  std::uint64_t x = sm(seed ^ sm(stream + 0x632be59bd9b4e019ULL)) + t * 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  x = x ^ (x >> 31);
  return static_cast<double>(x >> 11) * 0x1.0p-53;
}

struct Instance {
  DiscreteMeasure a, b;
  CostMatrix C;
  KernelMatrix K;
};

static Instance random_instance(std::size_t n, double eps, std::uint64_t seed) {
  PointList p;
  p.dim = 2;
  std::uint64_t t = 0;
  for (std::size_t k = 0; k < 2 * n; ++k) p.coords.push_back(draw(seed, 0, ++t));
  std::vector<double> wa(n), wb(n);
  double ta = 0, tb = 0;
  for (auto& x : wa) ta += (x = 0.2 + draw(seed, 0, ++t));
  for (auto& x : wb) tb += (x = 0.2 + draw(seed, 0, ++t));
  for (auto& x : wa) x /= ta;
  for (auto& x : wb) x /= tb;
  Instance inst;
  inst.C = sq_euclidean_cost(p, p);
  inst.K = kernel_from_cost(inst.C, eps);
  inst.a = new_measure(std::move(wa), p, true);
  inst.b = new_measure(std::move(wb), std::move(p), true);
  return inst;
}

static SolverConfig tight(double eps, double lambda = 0.0) {
  SolverConfig cfg;
  cfg.epsilon = eps;
  cfg.delta = 1e-13;
  cfg.max_iter = 200000;
  if (lambda > 0.0) cfg.lambda = lambda;
  return cfg;
}

int main() {
  run("two-atom OT closed form (test_solvers.cpp:60-73)", [] {
    auto sup = pts1d({0.0, 1.0});
    auto a = new_measure({0.5, 0.5}, sup, true);
    auto C = sq_euclidean_cost(sup, sup);
    auto K = kernel_from_cost(C, 1.0);
    auto res = sinkhorn_ot(K, a, a, tight(1.0));
    CHECK(res.report.converged);
    CHECK_CLOSE(res.plan.entry(0, 0), 0.36552928931500245, 1e-10);
    CHECK_CLOSE(res.plan.entry(0, 1), 0.13447071068499758, 1e-10);
    CHECK_CLOSE(ot_objective(res.plan, C, 1.0), -2.006408868078168, 1e-10);
  });
  run("three-atom OT (test_solvers.cpp:75-86)", [] {
    auto sup = pts1d({0.0, 0.3, 1.0});
    auto a = new_measure({0.2, 0.3, 0.5}, sup, true);
    auto b = new_measure({0.4, 0.4, 0.2}, sup, true);
    auto C = sq_euclidean_cost(sup, sup);
    auto K = kernel_from_cost(C, 0.5);
    auto res = sinkhorn_ot(K, a, b, tight(0.5));
    CHECK_CLOSE(res.plan.entry(0, 0), 0.1269550276492255, 1e-9);
    CHECK_CLOSE(ot_objective(res.plan, C, 0.5), -1.2371064921733375, 1e-10);
  });
  run("single-atom UOT fixed point (test_solvers.cpp:88-100)", [] {
    auto sup = pts1d({0.0});
    auto a = new_measure({2.0}, sup);
    auto b = new_measure({8.0}, sup);
    auto C = sq_euclidean_cost(sup, sup);
    auto K = kernel_from_cost(C, 1.0);
    CHECK(K.entries(0, 0) == 1.0);
    auto res = sinkhorn_uot(K, a, b, tight(1.0, 1.0));
    CHECK(std::abs(res.plan.entry(0, 0) - std::cbrt(16.0)) < 1e-8);
    CHECK_CLOSE(uot_objective(res.plan, C, a, b, 1.0, 1.0), 2.440473700630761, 1e-10);
  });
  run("two-atom UOT (test_solvers.cpp:102-115)", [] {
    auto sup = pts1d({0.0, 1.0});
    auto a = new_measure({0.7, 0.9}, sup);
    auto b = new_measure({0.4, 0.8}, sup);
    auto C = sq_euclidean_cost(sup, sup);
    auto K = kernel_from_cost(C, 0.5);
    auto res = sinkhorn_uot(K, a, b, tight(0.5, 2.0));
    CHECK_CLOSE(res.plan.entry(0, 0), 0.4880086699186626, 1e-9);
    CHECK_CLOSE(res.plan.entry(1, 1), 0.7835780682111341, 1e-9);
    CHECK_CLOSE(uot_objective(res.plan, C, a, b, 2.0, 0.5), -0.9506480667355813, 1e-9);
  });
  run("marginal residuals at delta=1e-10 (test_solvers.cpp:134-145)", [] {
    auto inst = random_instance(60, 0.3, 43);
    SolverConfig cfg = tight(0.3);
    cfg.delta = 1e-10;
    auto res = sinkhorn_ot(inst.K, inst.a, inst.b, cfg);
    CHECK(res.report.converged);
    CHECK(res.report.marginal_residual_row < 1e-6);
    CHECK(res.report.marginal_residual_col < 1e-6);
    auto rr = marginal_residuals(res.plan, inst.a, inst.b);
    CHECK_CLOSE(rr.first, res.report.marginal_residual_row, 1e-6);
    CHECK_CLOSE(rr.second, res.report.marginal_residual_col, 1e-6);
  });
  run("input validation (test_solvers.cpp:147-157)", [] {
    PointList p;
    p.dim = 2;
    p.coords = {0, 0, 1, 0, 0, 1, 1, 1, 0.5, 0.5};
    auto unnorm = new_measure({1, 1, 1, 1, 1}, p);
    auto C = sq_euclidean_cost(p, p);
    auto K = kernel_from_cost(C, 0.5);
    CHECK_THROWS_AS(sinkhorn_ot(K, unnorm, unnorm, tight(0.5)), NotNormalized);
    auto bal = random_instance(5, 0.5, 47);
    CHECK_THROWS_AS(sinkhorn_uot(bal.K, bal.a, bal.b, tight(0.5)), Error);
    auto small = random_instance(4, 0.5, 49);
    CHECK_THROWS_AS(sinkhorn_ot(bal.K, small.a, small.b, tight(0.5)), LengthMismatch);
  });
  run("log domain agrees with plain scaling (test_solvers.cpp:159-179)", [] {
    auto inst = random_instance(25, 0.2, 53);
    auto cfg = tight(0.2);
    auto plain = sinkhorn_ot(inst.K, inst.a, inst.b, cfg);
    cfg.stabilize = true;
    auto logd = sinkhorn_ot(inst.K, inst.a, inst.b, cfg);
    CHECK(logd.plan.log_domain);
    for (std::size_t i = 0; i < 25; ++i)
      for (std::size_t j = 0; j < 25; ++j) CHECK_CLOSE(logd.plan.entry(i, j), plain.plan.entry(i, j), 1e-6);
  });
  run("kl divergence (test_solvers.cpp:181-187)", [] {
    CHECK_CLOSE(kl_divergence({0.2, 0.0, 0.5}, {0.1, 0.3, 0.4}), 0.3502012117690939, 1e-14);
    CHECK_THROWS_AS(kl_divergence({0.5}, {0.0}), Error);
    CHECK_THROWS_AS(kl_divergence({0.5, 0.5}, {0.5}), LengthMismatch);
  });
  run("sparsified solver masks orphans; strict raises (test_solvers.cpp:189-204)", [] {
    auto inst = random_instance(80, 0.5, 59);
    SolverConfig cfg = tight(0.5);
    cfg.delta = 1e-8;
    auto res = spar_sink_ot(inst.K, inst.C, inst.a, inst.b, cfg, 240.0, 7);
    CHECK(res.plan.masked_rows > 0);
    CHECK(std::isfinite(res.report.objective));
    CHECK(res.report.sketch_nnz.has_value());
    SparSinkOptions strict;
    strict.strict = true;
    CHECK_THROWS_AS(spar_sink_ot(inst.K, inst.C, inst.a, inst.b, cfg, 240.0, 7, strict), DegenerateSketchError);
  });
  run("rand-sink switches the sampling law (test_solvers.cpp:206-216)", [] {
    auto inst = random_instance(40, 0.5, 61);
    SolverConfig cfg = tight(0.5);
    cfg.delta = 1e-8;
    SparSinkOptions uni;
    uni.probs = SketchProbs::Uniform;
    auto r1 = spar_sink_ot(inst.K, inst.C, inst.a, inst.b, cfg, 800.0, 3);
    auto r2 = spar_sink_ot(inst.K, inst.C, inst.a, inst.b, cfg, 800.0, 3, uni);
    CHECK(r1.report.sketch_nnz != r2.report.sketch_nnz);
  });
  run("theta shrinkage validated (test_solvers.cpp:218-230)", [] {
    auto inst = random_instance(40, 0.5, 67);
    SolverConfig cfg = tight(0.5);
    cfg.delta = 1e-8;
    SparSinkOptions opts;
    opts.theta = 0.3;
    auto res = spar_sink_ot(inst.K, inst.C, inst.a, inst.b, cfg, 700.0, 5, opts);
    CHECK(std::isfinite(res.report.objective));
    opts.theta = 1.0;
    CHECK_THROWS_AS(spar_sink_ot(inst.K, inst.C, inst.a, inst.b, cfg, 700.0, 5, opts), ThetaOutOfRange);
  });
  run("report serializes to json (test_solvers.cpp:232-239)", [] {
    auto inst = random_instance(10, 0.5, 71);
    auto res = sinkhorn_ot(inst.K, inst.a, inst.b, tight(0.5));
    res.report.objective = ot_objective(res.plan, inst.C, 0.5);
    const std::string j = res.report.to_json();
    CHECK(j.find("\"objective\"") != std::string::npos);
    CHECK(j.find("\"converged\": true") != std::string::npos);
  });
  run("ot probabilities (test_sparsify.cpp:51-61)", [] {
    auto sup = pts1d({0.0, 1.0});
    auto a = new_measure({0.25, 0.75}, sup, true);
    auto b = new_measure({0.5, 0.5}, sup, true);
    PointList p;
    p.dim = 2;
    for (int k = 1; k <= 4; ++k) p.coords.push_back(draw(3, 0, k));
    auto K = kernel_from_cost(sq_euclidean_cost(p, p), 1.0);
    auto plan = ot_probabilities(a, b, K);
    CHECK(plan.factorized_storage());
    CHECK_CLOSE(plan.prob(0, 0), 0.18301270189221933, 1e-14);
    CHECK_CLOSE(plan.prob(1, 1), 0.31698729810778065, 1e-14);
  });
  run("uot probabilities with 1/3 exponents (test_sparsify.cpp:63-81)", [] {
    auto sup = pts1d({0.0, 1.0});
    auto a = new_measure({0.3, 0.7}, sup);
    auto b = new_measure({0.4, 0.6}, sup);
    KernelMatrix K;
    K.epsilon = 1.0;
    K.entries = Matrix(2, 2);
    K.entries(0, 0) = 1.0;
    K.entries(0, 1) = 0.5;
    K.entries(1, 0) = 0.25;
    K.entries(1, 1) = 1.0;
    K.nnz_ratio = 1.0;
    auto plan = uot_probabilities(a, b, K, 1.0, 1.0);
    CHECK_CLOSE(plan.prob(0, 0), 0.2346093653249565, 1e-13);
    CHECK_CLOSE(plan.prob(0, 1), 0.2131567545016285, 1e-13);
    CHECK_CLOSE(plan.prob(1, 0), 0.19602777445115938, 1e-13);
    CHECK_CLOSE(plan.prob(1, 1), 0.35620610572225564, 1e-13);
  });
  run("sketch reproducible per seed, budget checks (test_sparsify.cpp:137-157)", [] {
    auto inst = random_instance(40, 0.5, 13);
    auto plan = ot_probabilities(inst.a, inst.b, inst.K);
    auto s1 = poisson_sparsify(inst.K, plan, 200.0, 42);
    auto s2 = poisson_sparsify(inst.K, plan, 200.0, 42);
    CHECK(s1.col_idx == s2.col_idx);
    CHECK(s1.values == s2.values);
    auto s3 = poisson_sparsify(inst.K, plan, 200.0, 43);
    CHECK(s1.col_idx != s3.col_idx);
    CHECK(static_cast<double>(s1.realized_nnz) < 200.0 + 5.0 * std::sqrt(200.0));
    CHECK_THROWS_AS(poisson_sparsify(inst.K, plan, 0.0, 1), BudgetTooLarge);
    CHECK_THROWS_AS(poisson_sparsify(inst.K, plan, 1600.0, 1), BudgetTooLarge);
  });
  run("spmv / spmv_t against the dense sketch (test_sparsify.cpp:186-211)", [] {
    auto inst = random_instance(30, 0.5, 19);
    auto plan = uniform_probabilities(inst.K);
    auto sk = poisson_sparsify(inst.K, plan, 300.0, 5);
    auto D = sk.to_dense();
    std::vector<double> v(30);
    for (int k = 0; k < 30; ++k) v[k] = draw(99, 0, k + 1);
    auto y = spmv(sk, v);
    auto yt = spmv_t(sk, v);
    for (std::size_t i = 0; i < 30; ++i) {
      double acc = 0, acct = 0;
      for (std::size_t j = 0; j < 30; ++j) {
        acc += D(i, j) * v[j];
        acct += D(j, i) * v[j];
      }
      CHECK_CLOSE(y[i], acc, 1e-12);
      CHECK_CLOSE(yt[i], acct, 1e-12);
    }
    std::vector<double> bad(31, 0.0);
    CHECK_THROWS_AS(spmv(sk, bad), LengthMismatch);
  });
  run("geometry (test_geometry.cpp:31-72)", [] {
    auto x = pts1d({0.0, 3.0});
    auto c2 = sq_euclidean_cost(x, x);
    CHECK(c2.entries(0, 1) == 9.0 && c2.c0 == 9.0);
    CHECK(euclidean_cost(x, x).entries(1, 0) == 3.0);
    PointList y;
    y.dim = 2;
    y.coords = {0.0, 0.0};
    CHECK_THROWS_AS(sq_euclidean_cost(x, y), DimensionMismatch);
    const double eta = 2.0;
    auto w = pts1d({0.0, 1.0, 3.14159265358979323846 * eta + 0.5});
    auto c = wfr_cost(w, w, eta);
    CHECK(c.entries(0, 0) == 0.0);
    CHECK_CLOSE(c.entries(0, 1), 0.06316210249493931, 1e-14);
    CHECK(std::isinf(c.entries(0, 2)));
    CHECK_THROWS_AS(wfr_cost(w, w, 0.0), NonPositiveEta);
    auto K = kernel_from_cost(wfr_cost(pts1d({0.0, 1.0, 100.0}), pts1d({0.0, 1.0, 100.0}), 2.0), 0.5);
    CHECK(K.entries(0, 2) == 0.0 && K.entries(0, 0) == 1.0);
    CHECK(std::abs(K.nnz_ratio - 5.0 / 9.0) < 1e-12);
    CHECK_THROWS_AS(kernel_from_cost(c, 0.0), NonPositiveEpsilon);
  });
  run("coordinate overload == dense drop-in (same sketch law, n^2-free)", [] {
    auto inst = random_instance(120, 0.05, 81);
    SolverConfig cfg = tight(0.05);
    cfg.delta = 1e-9;
    cfg.max_iter = 5000;
    auto dense = spar_sink_ot(inst.K, inst.C, inst.a, inst.b, cfg, 2000.0, 17);
    CostSpec cs;
    cs.scale = 1.0;
    auto coords = spar_sink_ot(inst.a.support, inst.b.support, cs, inst.a, inst.b, cfg, 2000.0, 17);
    CHECK(dense.report.sketch_nnz == coords.report.sketch_nnz);
    CHECK(dense.report.iterations == coords.report.iterations);
    CHECK_CLOSE(coords.report.objective, dense.report.objective, 1e-10);
  });
  run("batched frame pairs == one spar_sink_uot per pair (pairwise_wfr, harness.cpp:381-401)", [] {
    // 4 frames of 20x20 on [0,1]^2, WFR eta = 0.1, log domain, fp32 sketches
    const std::size_t side = 20, n = side * side;
    PointList grid;
    grid.dim = 2;
    for (std::size_t r = 0; r < side; ++r)
      for (std::size_t c = 0; c < side; ++c) {
        grid.coords.push_back(static_cast<double>(r) / (side - 1));
        grid.coords.push_back(static_cast<double>(c) / (side - 1));
      }
    std::vector<DiscreteMeasure> frames;
    for (int f = 0; f < 4; ++f) {
      std::vector<double> w(n);
      double t = 0.0;
      for (std::size_t i = 0; i < n; ++i) {
        const double dy = grid.coords[2 * i] - (0.3 + 0.1 * f), dx = grid.coords[2 * i + 1] - 0.5;
        t += (w[i] = 1e-4 + std::exp(-(dx * dx + dy * dy) / 0.02));
      }
      for (auto& x : w) x /= t;
      frames.push_back(new_measure(std::move(w), grid, true));
    }
    std::vector<std::pair<std::size_t, std::size_t>> pairs{{0, 1}, {0, 3}, {1, 2}, {2, 3}};
    std::vector<std::uint64_t> seeds{11, 12, 13, 14};
    SolverConfig cfg;
    cfg.epsilon = 0.01;
    cfg.lambda = 1.0;
    cfg.delta = 1e-6;
    cfg.max_iter = 400;
    cfg.stabilize = true;
    CostSpec cs;
    cs.kind = CostKind::WFR;
    cs.eta = 0.1;
    cs.scale = 1.0;
    SparSinkOptions o;
    o.values = ValuePrecision::F32;
    const double s = 10.0 * n * std::log(static_cast<double>(n));
    auto batch = spar_sink_uot_pairs(grid, cs, frames, pairs, cfg, s, seeds, o);
    CHECK(batch.size() == pairs.size());
    for (std::size_t k = 0; k < pairs.size(); ++k) {
      auto one = spar_sink_uot(grid, grid, cs, frames[pairs[k].first], frames[pairs[k].second], cfg, s, seeds[k], o);
      CHECK(!batch[k].failed);
      CHECK(batch[k].result.report.sketch_nnz == one.report.sketch_nnz);
      CHECK(std::abs(static_cast<long>(batch[k].result.report.iterations) - static_cast<long>(one.report.iterations)) <= 1);
      CHECK_CLOSE(batch[k].result.report.objective, one.report.objective, 1e-6);
      CHECK(batch[k].result.plan.log_domain && batch[k].result.plan.u.size() == n);
    }
    CHECK_THROWS_AS(spar_sink_uot_pairs(grid, cs, frames, pairs, cfg, s, {1, 2}, o), LengthMismatch);
  });
  run("sharded over the listed GPUs (SparSinkOptions::devices) == one-GPU solve", [] {
    auto inst = random_instance(400, 0.05, 91);
    SolverConfig cfg = tight(0.05);
    cfg.delta = -1.0;
    cfg.max_iter = 80;
    CostSpec cs;
    cs.scale = 1.0;
    auto one = spar_sink_ot(inst.a.support, inst.b.support, cs, inst.a, inst.b, cfg, 6000.0, 23);
    SparSinkOptions o;
    o.devices = {0};
    auto sh = spar_sink_ot(inst.a.support, inst.b.support, cs, inst.a, inst.b, cfg, 6000.0, 23, o);
    CHECK(one.report.sketch_nnz == sh.report.sketch_nnz);
    CHECK(one.report.iterations == sh.report.iterations);
    CHECK_CLOSE(sh.report.objective, one.report.objective, 1e-10);
    for (std::size_t i = 0; i < 400; ++i) CHECK_CLOSE(sh.plan.u[i], one.plan.u[i], 1e-10);
    // the failing rank's exception class crosses the multi-GPU driver
    DiscreteMeasure bad = inst.b;
    for (auto& w : bad.weights) w *= 2.0;
    bad.total_mass *= 2.0;
    CHECK_THROWS_AS(spar_sink_ot(inst.a.support, inst.b.support, cs, inst.a, bad, cfg, 6000.0, 23, o), NotNormalized);
  });
  std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
