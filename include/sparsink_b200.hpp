// sparsink_b200.hpp -- C++ drop-in for the reference's Spar-Sink entry points
// (namespace sparsink, proj/include/sparsink/*.hpp), implemented over the C ABI
// in spk.h (libsparsink_b200.so -> libspk_b200.so). Same names, argument
// meaning and exception classes; every O(n^2)/O(nnz) step runs on the B200.
//
// Reference declarations mirrored (proj/include/sparsink/):
//   errors.hpp:11-47     ErrorCategory, Error and its 18 classes
//   matrix.hpp:11-41     Matrix
//   measures.hpp:11-25   PointList, DiscreteMeasure, new_measure (measures.cpp:12-34)
//   geometry.hpp:10-34   CostKind, CostMatrix, KernelMatrix, sq_euclidean_cost,
//                        euclidean_cost, wfr_cost, kernel_from_cost
//   sparsify.hpp:14-98   PlanKind, SamplingPlan, SparseKernel, ot/uot/uniform_probabilities,
//                        shrink_with_uniform, poisson_sparsify, spmv, spmv_t
//   solvers.hpp:20-188   SolverConfig, EmptyPolicy, TransportPlan, SolveReport, SolveResult,
//                        sinkhorn_ot/uot (KernelMatrix, SparseKernel), SketchProbs,
//                        SparSinkOptions, spar_sink_ot/uot, ot_objective, uot_objective,
//                        marginal_residuals, kl_divergence, wfr_from_uot
// New (no n^2 host storage): CostSpec + coordinate overloads of spar_sink_ot/uot
// and sinkhorn_ot/uot (K recomputed on the fly), plus batched frame pairs.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "spk.h"

namespace sparsink {

// ---- errors (errors.hpp) --------------------------------------------------------
enum class ErrorCategory { Input = 4, DegenerateSketch = 3, Solver = 2 };

class Error : public std::runtime_error {
 public:
  Error(ErrorCategory cat, const std::string& msg) : std::runtime_error(msg), category_(cat) {}
  ErrorCategory category() const { return category_; }

 private:
  ErrorCategory category_;
};

#define SPARSINK_B200_ERROR(Name, Cat)                                              \
  class Name : public Error {                                                       \
   public:                                                                          \
    explicit Name(const std::string& msg) : Error(ErrorCategory::Cat, #Name ": " + msg) {} \
  }
SPARSINK_B200_ERROR(NegativeWeight, Input);
SPARSINK_B200_ERROR(LengthMismatch, Input);
SPARSINK_B200_ERROR(NotNormalized, Input);
SPARSINK_B200_ERROR(AllBlack, Input);
SPARSINK_B200_ERROR(EmptyOutput, Input);
SPARSINK_B200_ERROR(DimensionMismatch, Input);
SPARSINK_B200_ERROR(NonPositiveEta, Input);
SPARSINK_B200_ERROR(NonPositiveEpsilon, Input);
SPARSINK_B200_ERROR(DegenerateSupport, Input);
SPARSINK_B200_ERROR(AllZeroKernel, Input);
SPARSINK_B200_ERROR(ThetaOutOfRange, Input);
SPARSINK_B200_ERROR(BudgetTooLarge, Input);
SPARSINK_B200_ERROR(EmptyWindow, Input);
SPARSINK_B200_ERROR(InfiniteCostOnSupport, Input);
SPARSINK_B200_ERROR(IoError, Input);
SPARSINK_B200_ERROR(ZeroDenominator, Solver);
SPARSINK_B200_ERROR(BaselineFailed, Solver);
SPARSINK_B200_ERROR(DegenerateSketchError, DegenerateSketch);
#undef SPARSINK_B200_ERROR

// Device fault (no reference analogue): the CUDA path failed or no GPU exists.
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// ---- counter-based RNG (rng.hpp:10-50) ----------------------------------------------
// Draw t (t = 1, 2, ...) of stream (seed, stream) is the splitmix64 finalizer
// of mix_seed(seed, stream) + t * golden: any draw of any stream is addressable
// directly (the GPU sampler evaluates draw t of row i in closed form).
constexpr std::uint64_t kGoldenGamma = 0x9e3779b97f4a7c15ULL;
inline std::uint64_t splitmix64_finalize(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline std::uint64_t splitmix64(std::uint64_t x) { return splitmix64_finalize(x + kGoldenGamma); }
inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t stream) {
  return splitmix64(seed ^ splitmix64(stream + 0x632be59bd9b4e019ULL));
}

class CounterRng {
 public:
  explicit CounterRng(std::uint64_t seed, std::uint64_t stream = 0) : base_(mix_seed(seed, stream)) {}
  std::uint64_t next_u64() { return splitmix64_finalize(base_ + (++t_) * kGoldenGamma); }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }  // 53 bits in [0, 1)
  // Box-Muller, two draws per pair, the sine half kept for the next call (rng.cpp:7-21)
  double next_normal() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    const double u1 = std::max(next_double(), 1e-300), u2 = next_double();
    const double r = std::sqrt(-2.0 * std::log(u1)), th = 2.0 * 3.14159265358979323846 * u2;
    spare_ = r * std::sin(th);
    spare_ok_ = true;
    return r * std::cos(th);
  }

 private:
  std::uint64_t base_;
  std::uint64_t t_ = 0;
  bool spare_ok_ = false;
  double spare_ = 0.0;
};

// ---- containers ---------------------------------------------------------------------
class Matrix {
 public:
  Matrix() = default;
  Matrix(std::size_t rows, std::size_t cols, double fill = 0.0) : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  double& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
  double operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
  double* row(std::size_t i) { return data_.data() + i * cols_; }
  const double* row(std::size_t i) const { return data_.data() + i * cols_; }
  std::vector<double>& data() { return data_; }
  const std::vector<double>& data() const { return data_; }

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

struct PointList {
  std::vector<double> coords;
  std::size_t dim = 0;
  std::size_t size() const { return dim == 0 ? 0 : coords.size() / dim; }
  const double* point(std::size_t i) const { return coords.data() + i * dim; }
};

struct DiscreteMeasure {
  std::vector<double> weights;
  PointList support;
  double total_mass = 0.0;
  std::size_t size() const { return weights.size(); }
};

DiscreteMeasure new_measure(std::vector<double> weights, PointList support, bool require_simplex = false);

enum class CostKind { SqEuclidean, Euclidean, WFR };

struct CostMatrix {
  Matrix entries;
  CostKind kind = CostKind::SqEuclidean;
  double eta = 0.0;
  double c0 = 0.0;
};

struct KernelMatrix {
  Matrix entries;
  double epsilon = 0.0;
  double nnz_ratio = 1.0;
  std::size_t size() const { return entries.rows(); }
};

CostMatrix sq_euclidean_cost(const PointList& x, const PointList& y);
CostMatrix euclidean_cost(const PointList& x, const PointList& y);
CostMatrix wfr_cost(const PointList& x, const PointList& y, double eta);
KernelMatrix kernel_from_cost(const CostMatrix& cost, double epsilon);
// WFR eta whose cut pi * eta keeps the target fraction of the n^2 pairwise
// distances (geometry.cpp:104-135).
double eta_for_sparsity(const PointList& x, double target_nnz_ratio);

// ---- sketches ---------------------------------------------------------------------------
enum class PlanKind { OT, UOT, Barycenter, Uniform };

// A sampling plan is a recipe evaluated on the device: kind, marginals,
// lambda/epsilon and theta; prob(i, j) asks the device (SamplingPlan::prob).
class SamplingPlan {
 public:
  double prob(std::size_t i, std::size_t j) const;
  std::size_t size() const { return kernel_ ? kernel_->size() : 0; }
  PlanKind kind() const { return kind_; }
  double theta() const { return theta_; }
  bool factorized_storage() const;

  friend SamplingPlan ot_probabilities(const DiscreteMeasure&, const DiscreteMeasure&, const KernelMatrix&);
  friend SamplingPlan uot_probabilities(const DiscreteMeasure&, const DiscreteMeasure&, const KernelMatrix&, double,
                                        double);
  friend SamplingPlan uniform_probabilities(const KernelMatrix&);
  friend SamplingPlan barycenter_probabilities(const DiscreteMeasure&, const KernelMatrix&);
  friend SamplingPlan shrink_with_uniform(const SamplingPlan&, double);
  friend struct PlanAccess;

 private:
  PlanKind kind_ = PlanKind::Uniform;
  const KernelMatrix* kernel_ = nullptr;
  std::vector<double> a_, b_;
  double lambda_ = 0.0, epsilon_ = 1.0, theta_ = 0.0;
};

struct SparseKernel {
  std::vector<std::size_t> row_ptr;
  std::vector<std::uint32_t> col_idx;
  std::vector<double> values;
  std::size_t n = 0;
  std::uint64_t seed = 0;
  std::size_t realized_nnz = 0;
  double epsilon = 0.0;
  std::size_t size() const { return n; }
  Matrix to_dense() const;
};

SamplingPlan ot_probabilities(const DiscreteMeasure& a, const DiscreteMeasure& b, const KernelMatrix& K);
SamplingPlan uot_probabilities(const DiscreteMeasure& a, const DiscreteMeasure& b, const KernelMatrix& K,
                               double lambda, double epsilon);
SamplingPlan uniform_probabilities(const KernelMatrix& K);
// Spar-IBP's column plan for kernel k: rows 1/n, columns sqrt(b_k) normalised,
// masked to the support (sparsify.cpp:117-135).
SamplingPlan barycenter_probabilities(const DiscreteMeasure& b_k, const KernelMatrix& K_k);
SamplingPlan shrink_with_uniform(const SamplingPlan& plan, double theta);
SparseKernel poisson_sparsify(const KernelMatrix& K, const SamplingPlan& plan, double s, std::uint64_t seed);
std::vector<double> spmv(const SparseKernel& M, const std::vector<double>& v);
std::vector<double> spmv_t(const SparseKernel& M, const std::vector<double>& u);

// ---- solvers ------------------------------------------------------------------------------
struct SolverConfig {
  double epsilon = 1.0;
  double lambda = std::numeric_limits<double>::infinity();
  double delta = 1e-6;
  std::size_t max_iter = 1000;
  bool stabilize = false;
};

enum class EmptyPolicy { Error, Mask };

struct TransportPlan {
  std::vector<double> u, v;
  std::vector<double> log_u, log_v;
  bool log_domain = false;
  const KernelMatrix* dense_kernel = nullptr;
  const SparseKernel* sparse_kernel = nullptr;
  bool converged = false;
  std::size_t iterations = 0;
  std::size_t masked_rows = 0;
  std::size_t masked_cols = 0;

  std::size_t size() const { return u.size(); }
  double scaling_u(std::size_t i) const { return log_domain ? std::exp(log_u[i]) : u[i]; }
  double scaling_v(std::size_t j) const { return log_domain ? std::exp(log_v[j]) : v[j]; }
  double entry(std::size_t i, std::size_t j) const;
  std::vector<double> row_marginal() const;
  std::vector<double> col_marginal() const;
};

struct SolveReport {
  double objective = std::numeric_limits<double>::quiet_NaN();
  std::size_t iterations = 0;
  double marginal_residual_row = 0.0;
  double marginal_residual_col = 0.0;
  double wall_time_s = 0.0;
  std::optional<std::size_t> sketch_nnz;
  bool converged = false;
  bool diverged = false;
  std::uint64_t seed = 0;
  double kernel_mean = 0.0;
  std::string to_json() const;
};

struct SolveResult {
  TransportPlan plan;
  SolveReport report;
};

template <class Kernel>
SolveResult sinkhorn_ot(const Kernel& K, const DiscreteMeasure& a, const DiscreteMeasure& b, const SolverConfig& cfg,
                        EmptyPolicy empty_policy = EmptyPolicy::Error);
template <class Kernel>
SolveResult sinkhorn_uot(const Kernel& K, const DiscreteMeasure& a, const DiscreteMeasure& b, const SolverConfig& cfg,
                         EmptyPolicy empty_policy = EmptyPolicy::Error);

template <>
SolveResult sinkhorn_ot<KernelMatrix>(const KernelMatrix&, const DiscreteMeasure&, const DiscreteMeasure&,
                                      const SolverConfig&, EmptyPolicy);
template <>
SolveResult sinkhorn_uot<KernelMatrix>(const KernelMatrix&, const DiscreteMeasure&, const DiscreteMeasure&,
                                       const SolverConfig&, EmptyPolicy);
template <>
SolveResult sinkhorn_ot<SparseKernel>(const SparseKernel&, const DiscreteMeasure&, const DiscreteMeasure&,
                                      const SolverConfig&, EmptyPolicy);
template <>
SolveResult sinkhorn_uot<SparseKernel>(const SparseKernel&, const DiscreteMeasure&, const DiscreteMeasure&,
                                       const SolverConfig&, EmptyPolicy);

enum class SketchProbs { Importance, Uniform };

// Storage of the sketch values K~ on the device (B200 extension; the
// reference's SparseKernel is fp64). F32 halves the loop's value stream
// (configs 3 and 4); sums and scalings stay fp64.
enum class ValuePrecision { F64, F32 };

struct SparSinkOptions {
  double theta = 0.0;
  SketchProbs probs = SketchProbs::Importance;
  bool strict = false;
  ValuePrecision values = ValuePrecision::F64;  // B200 extension
  // B200 extension: GPUs of this process for the coordinate overloads of
  // spar_sink_*. Empty = the thread's device (set_device). Listed: the sketch's
  // rows and columns are sharded over them (NCCL inside the library, one
  // driver thread per GPU, spk_spar_sink_multi).
  std::vector<int> devices;
};

SolveResult spar_sink_ot(const KernelMatrix& K, const CostMatrix& C, const DiscreteMeasure& a,
                         const DiscreteMeasure& b, const SolverConfig& cfg, double s, std::uint64_t seed,
                         const SparSinkOptions& opts = {});
SolveResult spar_sink_uot(const KernelMatrix& K, const CostMatrix& C, const DiscreteMeasure& a,
                          const DiscreteMeasure& b, const SolverConfig& cfg, double s, std::uint64_t seed,
                          const SparSinkOptions& opts = {});

double ot_objective(const TransportPlan& T, const CostMatrix& C, double epsilon);
double uot_objective(const TransportPlan& T, const CostMatrix& C, const DiscreteMeasure& a, const DiscreteMeasure& b,
                     double lambda, double epsilon);
std::pair<double, double> marginal_residuals(const TransportPlan& T, const DiscreteMeasure& a,
                                             const DiscreteMeasure& b);
double kl_divergence(const std::vector<double>& x, const std::vector<double>& y);
inline double wfr_from_uot(double uot_value) { return std::sqrt(std::max(uot_value, 0.0)); }

// ---- new: coordinate overloads (no n^2 host storage) ----------------------------------------
struct CostSpec {
  CostKind kind = CostKind::SqEuclidean;
  double eta = 0.0;    // WFR cut-off scale
  double scale = 0.0;  // C = cost / scale; <= 0 divides by c0 = max finite cost
};

// Spar-Sink with costs/kernels recomputed from x, y on the device. The report
// carries the objective; the plan holds u, v (no kernel pointer: the sketch
// lives and dies on the device, as in spar_sink_*).
SolveResult spar_sink_ot(const PointList& x, const PointList& y, const CostSpec& cost, const DiscreteMeasure& a,
                         const DiscreteMeasure& b, const SolverConfig& cfg, double s, std::uint64_t seed,
                         const SparSinkOptions& opts = {});
SolveResult spar_sink_uot(const PointList& x, const PointList& y, const CostSpec& cost, const DiscreteMeasure& a,
                          const DiscreteMeasure& b, const SolverConfig& cfg, double s, std::uint64_t seed,
                          const SparSinkOptions& opts = {});
// Dense Sinkhorn with K recomputed on the fly every iteration (config-5 comparator).
SolveResult sinkhorn_ot(const PointList& x, const PointList& y, const CostSpec& cost, const DiscreteMeasure& a,
                        const DiscreteMeasure& b, const SolverConfig& cfg, EmptyPolicy empty_policy = EmptyPolicy::Error);
SolveResult sinkhorn_uot(const PointList& x, const PointList& y, const CostSpec& cost, const DiscreteMeasure& a,
                         const DiscreteMeasure& b, const SolverConfig& cfg, EmptyPolicy empty_policy = EmptyPolicy::Error);

// Batched frame pairs (config 3; the per-pair spar_sink_uot calls of
// pairwise_wfr, harness.cpp:381-401): pair k solves
//   spar_sink_uot(support, support, cost, measures[pairs[k].first],
//                 measures[pairs[k].second], cfg, s, seeds[k], opts)
// with every sketch drawn by one device batch and, in the log domain
// (cfg.stabilize), every loop run by one batched launch (a cluster of CTAs per
// pair). A pair whose solve fails gets failed = true, its exception class in
// error, and a NaN objective -- the reference's NaN distance and failed_pairs
// count; the other pairs complete. Results come in pair order.
struct PairSolve {
  SolveResult result;
  bool failed = false;
  std::string error;
};
std::vector<PairSolve> spar_sink_uot_pairs(const PointList& support, const CostSpec& cost,
                                           const std::vector<DiscreteMeasure>& measures,
                                           const std::vector<std::pair<std::size_t, std::size_t>>& pairs,
                                           const SolverConfig& cfg, double s, const std::vector<std::uint64_t>& seeds,
                                           const SparSinkOptions& opts = {});

// Runtime controls of the device context used by this thread.
void set_device(int device);
void set_deterministic(bool on);  // reference summation order (bit-identical OT scalings)

}  // namespace sparsink
