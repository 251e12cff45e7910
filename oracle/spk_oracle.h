/*
 * spk_oracle.h -- CPU restatement of the Spar-Sink hot path (TEST INFRASTRUCTURE).
 *
 * This is the CHECKER, not the product. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The
 * product path (paper_2306_06581_b200/) never links or calls it.
 *
 * Every function restates one reference function; the citation is the
 * reference file:line (relative to /root/reference/proj) it follows.
 * Arithmetic order is kept sequential and contraction-free (compile with
 * -O2 -ffp-contract=off, no -march) so that, like the reference built with
 * its own -O2 flags on x86-64, no FMA is formed.
 *
 * Pinning: tests/test_oracle_golden.py checks this restatement against the
 * reference's own known-answer values (tests/test_sparsify.cpp,
 * tests/test_solvers.cpp, tests/test_geometry.cpp) and, when oracle/_ref is
 * built, bit-for-bit against the compiled reference (sketch index sets,
 * values, scalings, iteration counts).
 */
#ifndef SPK_ORACLE_H_
#define SPK_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error kinds: same numbering as include/spk.h (SPK_E_*). 0 = ok. */
enum {
  SPKO_OK = 0,
  SPKO_E_ERROR = 1, /* plain sparsink::Error with a category */
  SPKO_E_NEGATIVE_WEIGHT = 2,
  SPKO_E_LENGTH_MISMATCH = 3,
  SPKO_E_NOT_NORMALIZED = 4,
  SPKO_E_DIMENSION_MISMATCH = 7,
  SPKO_E_NON_POSITIVE_ETA = 8,
  SPKO_E_NON_POSITIVE_EPSILON = 9,
  SPKO_E_ALL_ZERO_KERNEL = 11,
  SPKO_E_THETA_OUT_OF_RANGE = 12,
  SPKO_E_BUDGET_TOO_LARGE = 13,
  SPKO_E_INFINITE_COST_ON_SUPPORT = 15,
  SPKO_E_ZERO_DENOMINATOR = 17,
  SPKO_E_DEGENERATE_SKETCH = 19,
};

enum { SPKO_COST_SQEUCLID = 0, SPKO_COST_EUCLID = 1, SPKO_COST_WFR = 2 };
enum { SPKO_PLAN_OT = 0, SPKO_PLAN_UOT = 1, SPKO_PLAN_BARY = 2, SPKO_PLAN_UNIFORM = 3 };
enum { SPKO_POLICY_ERROR = 0, SPKO_POLICY_MASK = 1 };

/* ---- RNG: proj/include/sparsink/rng.hpp ---------------------------------- */
uint64_t spko_splitmix64(uint64_t x);                    /* rng.hpp:10-15 */
uint64_t spko_mix_seed(uint64_t seed, uint64_t stream);  /* rng.hpp:17-19 */
/* t-th (1-based) next_double of CounterRng(seed, stream): rng.hpp:24-40 */
double spko_counter_draw(uint64_t seed, uint64_t stream, uint64_t t);
/* count successive next_double() of CounterRng(seed, stream) */
void spko_rng_doubles(uint64_t seed, uint64_t stream, int64_t count, double* out);
/* count successive next_normal() (Box-Muller with spare), rng.cpp:7-21 */
void spko_rng_normals(uint64_t seed, uint64_t stream, int64_t count, double* out);

/* ---- measures: proj/src/measures.cpp:12-34 -------------------------------- */
/* Validates weights (>=0, finite, not all zero, optional simplex), returns
 * the sequential total in *total. */
int spko_new_measure(const double* w, int64_t n, int require_simplex, double* total);

/* ---- geometry: proj/src/geometry.cpp -------------------------------------- */
/* One cost entry exactly as pairwise_cost computes it (geometry.cpp:16-66). */
double spko_cost_entry(const double* p, const double* q, int dim, int kind, double eta);
/* Dense n_x x n_y cost + c0 (max finite entry); geometry.cpp:25-66. */
int spko_pairwise_cost(const double* x, int64_t nx, const double* y, int64_t ny,
                       int dim, int kind, double eta, double* C, double* c0);
/* K = isinf(C) ? 0 : exp(-C/eps); nnz_ratio; geometry.cpp:83-102. */
int spko_kernel_from_cost(const double* C, int64_t rows, int64_t cols, double eps,
                          double* K, double* nnz_ratio);

/* ---- sampling plans: proj/src/sparsify.cpp:71-167, sparsify.hpp:20-54 ---- */
typedef struct {
  int kind;
  int64_t n;
  int factorized;      /* 1: p = row_w[i]*col_w[j]; 0: grid */
  double theta;        /* lazy theta (factorized only) */
  int64_t kernel_nnz;
  double* grid;        /* n*n, owned, or NULL */
  double* row_w;       /* n, owned, or NULL */
  double* col_w;
} spko_plan;

void spko_plan_free(spko_plan* p);
double spko_plan_prob(const spko_plan* p, int64_t i, int64_t j); /* sparsify.hpp:28-34 */
int spko_ot_probabilities(const double* a, const double* b, int64_t n, const double* K,
                          double nnz_ratio, spko_plan* out);          /* sparsify.cpp:71-91 */
int spko_uot_probabilities(const double* a, const double* b, int64_t n, const double* K,
                           double nnz_ratio, double lambda, double eps,
                           spko_plan* out);                             /* :93-115 */
int spko_uniform_probabilities(int64_t n, const double* K, double nnz_ratio,
                               spko_plan* out);                         /* :137-147 */
int spko_shrink_with_uniform(spko_plan* p, double theta);               /* :149-167 */

/* ---- sketch: proj/src/sparsify.cpp:169-226 -------------------------------- */
typedef struct {
  int64_t n;
  int64_t nnz;
  int64_t* row_ptr;   /* n+1 */
  uint32_t* col_idx;  /* nnz */
  double* values;     /* nnz */
} spko_csr;

void spko_csr_free(spko_csr* s);
int spko_poisson_sparsify(const double* K, int64_t n, const spko_plan* plan, double s,
                          uint64_t seed, spko_csr* out);                /* :169-201 */
void spko_spmv(const spko_csr* M, const double* v, double* out);        /* :203-213 */
void spko_spmv_t(const spko_csr* M, const double* u, double* out);      /* :215-226 */

/* Coordinate-based restatement of poisson_sparsify for a ROW SUBSET, used
 * where the reference cannot hold dense K (config 4, n = 1e6). Same draw
 * addressing (stream (seed, i), one draw per nonzero-K entry), kernel
 * computed per entry as kernel_from_cost(cost/scale, eps) would. The plan is
 * passed in already normalised: p = (row_w[i]*col_w[j])*inv (grid) or
 * row_w[i]*col_w[j] (factorized, inv ignored), or for UOT
 * ((row_w[i]*col_w[j])*pow(K, g_k))*inv. Output rows are [r0, r1). */
int spko_sample_rows_coords(const double* x, const double* y, int64_t n, int dim,
                            int cost_kind, double eta, double scale, double eps,
                            int plan_kind, int factorized, const double* row_w,
                            const double* col_w, double g_k, double inv,
                            double s, uint64_t seed, int64_t r0, int64_t r1,
                            spko_csr* out);

/* ---- solvers: proj/include/sparsink/solvers.hpp, proj/src/solvers.cpp ---- */
typedef struct {
  double epsilon, lambda, delta;
  int64_t max_iter;
  int stabilize;
} spko_cfg;

typedef struct {
  int64_t iterations;
  int converged, diverged, log_domain;
  int64_t masked_rows, masked_cols;
  double residual_row, residual_col;
  double kernel_mean;
} spko_result;

/* sinkhorn_ot / sinkhorn_uot (solvers.hpp:209-232) on a sketch (SparseKernel)
 * or dense K (KernelMatrix, K != NULL, sk == NULL). uot=0: OT with the
 * simplex check; uot=1: exponent lambda/(lambda+eps). u, v (and log_u,
 * log_v when non-NULL and the log-domain path ran) receive the scalings.
 * On error returns the kind; msg (if non-NULL, len bytes) gets the text. */
int spko_sinkhorn(const spko_csr* sk, const double* K, int64_t n, const double* a,
                  const double* b, double a_total, double b_total, const spko_cfg* cfg,
                  int policy, int uot, double* u, double* v, double* log_u,
                  double* log_v, spko_result* res, char* msg, size_t len);

/* Bare loop of time_scaling_iters (harness.cpp:262-278): iters of
 * u = tmp>0 ? a/tmp : 0, v = ... with no guards. Returns seconds/iter. */
double spko_time_scaling_iters(const spko_csr* sk, const double* a, const double* b,
                               int64_t iters, double* u, double* v);

/* Plan readout over the sketch support (solvers.hpp:234-252,
 * solvers.cpp:195-225,246-308). Cost entries come from dense C (n*n) when
 * C != NULL, else are recomputed from coordinates x, y (dim, kind, eta,
 * divided by scale). Writes row/col marginals (n each, may be NULL) and
 * the objective (OT: uot=0; UOT: uot=1 with lambda). log_u/log_v are used
 * when log_domain != 0. */
int spko_readout(const spko_csr* sk, const double* K, int64_t n, const double* u,
                 const double* v, const double* log_u, const double* log_v,
                 int log_domain, const double* C, const double* x, const double* y,
                 int dim, int cost_kind, double eta, double scale, const double* a,
                 const double* b, int uot, double lambda, double eps, double* row_m,
                 double* col_m, double* objective, char* msg, size_t len);

/* kl_divergence (solvers.cpp:246-260). */
int spko_kl_divergence(const double* x, const double* y, int64_t n, double* out);

/* Spar-Sink end to end on dense K, C (solvers.cpp:314-378): plan ->
 * [theta] -> sample -> [strict coverage] -> loop (Mask unless strict) ->
 * objective. probs: 0 importance, 1 uniform (Rand-Sink). The sketch is
 * returned in *sk_out when non-NULL (caller frees). */
int spko_spar_sink(const double* K, double nnz_ratio, const double* C, int64_t n,
                   const double* a, const double* b, double a_total, double b_total,
                   const spko_cfg* cfg, double s, uint64_t seed, double theta, int probs,
                   int strict, int uot, double* u, double* v, double* log_u, double* log_v,
                   spko_result* res, double* objective, int64_t* sketch_nnz,
                   spko_csr* sk_out, char* msg, size_t len);

#ifdef __cplusplus
}
#endif

#endif /* SPK_ORACLE_H_ */
