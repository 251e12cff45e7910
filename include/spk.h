/*
 * spk.h -- C ABI of the B200-native Spar-Sink hot path (libspk_b200.so).
 *
 * Plain pointers and sizes only; no CUDA, C++ or torch types cross this
 * boundary. Every entry point blocks until its host outputs are written,
 * never throws, and returns 0 or the reference's ErrorCategory value
 * (proj/include/sparsink/errors.hpp:11): 2 = solver, 3 = degenerate sketch,
 * 4 = input, plus 5 = CUDA/device fault. spk_last_error() then reports the
 * exception class (SPK_E_*) and the reference-style message
 * ("<Class>: text", errors.hpp:23-28) so a C++ shim can rethrow the SAME
 * type (see include/sparsink_b200.hpp and INTEGRATION.md).
 *
 * Reference interfaces replaced (relative to /root/reference/proj):
 *   spk_spar_sink          spar_sink_ot / spar_sink_uot   include/sparsink/solvers.hpp:159-167
 *                          (+ coordinate overload, no n^2 host storage)
 *   spk_sinkhorn           sinkhorn_ot / sinkhorn_uot<KernelMatrix>   solvers.hpp:137-147,209-232
 *   spk_sketch_solve       sinkhorn_ot / sinkhorn_uot<SparseKernel>   solvers.hpp:137-147
 *   spk_sketch_build       ot/uot/uniform_probabilities + shrink_with_uniform
 *                          + poisson_sparsify            include/sparsink/sparsify.hpp:74-95
 *   spk_sketch_spmv        spmv / spmv_t                  sparsify.hpp:97-98
 *   spk_sketch_readout     ot_objective / uot_objective / marginal_residuals /
 *                          TransportPlan::row_marginal,col_marginal  solvers.hpp:53-54,170-181
 *   spk_plan_probs         SamplingPlan::prob on a set of (i, j)     sparsify.hpp:28-34
 *   spk_cost_kernel        sq_euclidean_cost / euclidean_cost / wfr_cost +
 *                          kernel_from_cost               include/sparsink/geometry.hpp:28-36
 */
#ifndef SPK_H_
#define SPK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPK_ABI_VERSION 1

/* ---- status and error classes --------------------------------------------- */
enum spk_status {
  SPK_OK = 0,
  SPK_STATUS_SOLVER = 2,            /* ErrorCategory::Solver */
  SPK_STATUS_DEGENERATE_SKETCH = 3, /* ErrorCategory::DegenerateSketch */
  SPK_STATUS_INPUT = 4,             /* ErrorCategory::Input */
  SPK_STATUS_DEVICE = 5             /* CUDA fault / missing device (no reference analogue) */
};

/* Exception classes of errors.hpp:30-47 (plus the plain Error base). */
enum spk_error_kind {
  SPK_E_NONE = 0,
  SPK_E_ERROR = 1, /* sparsink::Error(category, msg) */
  SPK_E_NEGATIVE_WEIGHT = 2,
  SPK_E_LENGTH_MISMATCH = 3,
  SPK_E_NOT_NORMALIZED = 4,
  SPK_E_ALL_BLACK = 5,
  SPK_E_EMPTY_OUTPUT = 6,
  SPK_E_DIMENSION_MISMATCH = 7,
  SPK_E_NON_POSITIVE_ETA = 8,
  SPK_E_NON_POSITIVE_EPSILON = 9,
  SPK_E_DEGENERATE_SUPPORT = 10,
  SPK_E_ALL_ZERO_KERNEL = 11,
  SPK_E_THETA_OUT_OF_RANGE = 12,
  SPK_E_BUDGET_TOO_LARGE = 13,
  SPK_E_EMPTY_WINDOW = 14,
  SPK_E_INFINITE_COST_ON_SUPPORT = 15,
  SPK_E_IO_ERROR = 16,
  SPK_E_ZERO_DENOMINATOR = 17,
  SPK_E_BASELINE_FAILED = 18,
  SPK_E_DEGENERATE_SKETCH_ERROR = 19,
  SPK_E_DEVICE = 20
};

/* ---- enums mirroring the reference ---------------------------------------- */
enum spk_cost_kind { SPK_COST_SQEUCLID = 0, SPK_COST_EUCLID = 1, SPK_COST_WFR = 2 }; /* geometry.hpp:10 */
enum spk_plan_kind { SPK_PLAN_OT = 0, SPK_PLAN_UOT = 1, SPK_PLAN_BARYCENTER = 2, SPK_PLAN_UNIFORM = 3 }; /* sparsify.hpp:14 */
enum spk_empty_policy { SPK_POLICY_ERROR = 0, SPK_POLICY_MASK = 1 };  /* solvers.hpp:32 */
enum spk_probs { SPK_PROBS_IMPORTANCE = 0, SPK_PROBS_UNIFORM = 1 };   /* solvers.hpp:149 */
enum spk_value_type { SPK_VALUES_F64 = 0, SPK_VALUES_F32 = 1 };

/* ---- plain structs ---------------------------------------------------------- */

/* The Gibbs kernel and its cost, in one of two forms.
 * Dense form (KernelMatrix + CostMatrix, geometry.hpp:13-26): K != NULL,
 *   n*n row-major host fp64; nnz_ratio as KernelMatrix::nnz_ratio; C may be
 *   NULL when no objective is needed. Cost-only form (K == NULL, C != NULL,
 *   x == NULL): costs for a readout over a sketch.
 * Coordinate form (new; no n^2 storage): K == NULL, x and y are n*dim
 *   row-major host fp64 points; C_ij = cost(x_i, y_j) / cost_scale computed
 *   exactly as pairwise_cost (geometry.cpp:16-66) and the caller's division;
 *   cost_scale <= 0 means "divide by c0 = max finite cost" (the configs'
 *   max-normalisation); K_ij = isinf(C) ? 0 : exp(-C_ij / kernel_epsilon)
 *   (kernel_from_cost, geometry.cpp:83-102). */
typedef struct {
  int64_t n;
  const double* K;
  double nnz_ratio;
  const double* C;
  const double* x;
  const double* y;
  int32_t dim;
  int32_t cost_kind;
  double eta;
  double cost_scale;
  double kernel_epsilon;
} spk_kernel_desc;

/* SolverConfig (solvers.hpp:20-26) + the EmptyPolicy argument. */
typedef struct {
  double epsilon;
  double lambda; /* +INFINITY = balanced */
  double delta;
  int64_t max_iter;
  int32_t stabilize;    /* log-domain iterations */
  int32_t empty_policy; /* spk_empty_policy */
} spk_solver_cfg;

/* SparSinkOptions (solvers.hpp:151-157) + storage choice. */
typedef struct {
  double theta;
  int32_t probs;      /* spk_probs */
  int32_t strict;
  int32_t value_type; /* spk_value_type: sketch values fp64 (default) or fp32 */
  int32_t reserved;
} spk_sketch_opts;

/* SolveReport (solvers.hpp:61-76) + TransportPlan flags (:40-43) + phase
 * timings measured with CUDA events on the context's stream. */
typedef struct {
  double objective;
  int64_t iterations;
  double residual_row;
  double residual_col;
  double wall_time_s;
  int64_t sketch_nnz; /* -1 when no sketch (dense solve) */
  int32_t converged;
  int32_t diverged;
  uint64_t seed;
  double kernel_mean;
  int64_t masked_rows;
  int64_t masked_cols;
  int32_t log_domain;
  int32_t factorized_plan;
  int64_t kernel_nnz;
  double t_plan_s;
  double t_sample_s;
  double t_loop_s;
  double t_readout_s;
} spk_report;

typedef struct spk_ctx spk_ctx;
typedef struct spk_sketch spk_sketch;

/* ---- context ---------------------------------------------------------------- */
int spk_ctx_create(int device, spk_ctx** out);
void spk_ctx_destroy(spk_ctx* ctx);
/* Use an external CUDA stream (a cudaStream_t passed as void*; NULL = the
 * context's own stream). Lets callers time kernels on their stream. */
int spk_ctx_set_stream(spk_ctx* ctx, void* stream);
void* spk_ctx_stream(spk_ctx* ctx);
/* Option keys. SPK_OPT_DETERMINISTIC=1 selects the parity kernels: one thread
 * per output summing in the reference's index order with no FMA, and
 * sequential residual sums, so OT scalings and iteration counts are
 * bit-identical to the CPU reference on the same sketch. */
enum spk_option {
  SPK_OPT_DETERMINISTIC = 1,
  SPK_OPT_LOOP_BLOCKS_PER_SM = 2,
  SPK_OPT_OTF_FP32 = 3,      /* dense on-the-fly comparator: K in fp32 (1) or fp64 (0) */
  SPK_OPT_BLOCKED_LOOP = 4,  /* fast sparse loop: slab x block layout (1), CSR/CSC (0), auto (2, default: n >= 2^17 always;
                                2^15 <= n < 2^17 once a sketch is solved again or max_iter >= 400; chunk padding <= 80%) */
  SPK_OPT_BLOCKED_MAX_W = 5, /* cap on the staged tile width (testing) */
  SPK_OPT_TWO_PASS_SAMPLER = 6, /* sampler: always the exact two-pass kernels (testing) */
  SPK_OPT_BLOCKED_SPLIT = 7,    /* slab x block loop: column parts per row slab (0 auto, 1, 2 = CTA pairs) */
  SPK_OPT_BLOCKED_SPREAD = 8,   /* slab x block layout, chunk placement: 1 (default) edge colouring of the accumulator / x bank
                                   classes, 2 greedy column dealing, 0 plain run placement */
  SPK_OPT_BLOCKED_CLUSTER = 9,  /* slab x block loop: CTA pairs as 2-CTA clusters sharing partial sums (1, default, when they fit) */
  SPK_OPT_BATCH_CLUSTER = 10,   /* batched log loop: CTAs (SMs) per sketch as one cluster: 1, 2 (default) or 4 */
  SPK_OPT_BATCH_UNROLL = 11,    /* batched log loop: entry loads in flight per lane: 4 or 8 (default) */
  SPK_OPT_SMALL_LOOP = 12,      /* fast mode, small sketches: the loop on ONE cluster with the scalings in
                                   shared memory (1, default) or the persistent grid loop (0) */
  SPK_OPT_SMALL_CLUSTER = 13,   /* that cluster's size: 16 (default, non-portable), 8, 4, 2, 1 */
  SPK_OPT_SMALL_MAX_NNZ = 14,   /* largest sketch (entries) it takes (default 4e6) */
  SPK_OPT_ROW_LANES = 15        /* grid loop, fast mode: lanes per sketch row: 0 auto (8 when rows average <= 256
                                   entries: 4 rows in flight per warp), 8, 32 */
};
int spk_ctx_set_option(spk_ctx* ctx, int key, int64_t value);
/* Current value of an option key (SPK_STATUS_INPUT for an unknown key). */
int spk_ctx_get_option(const spk_ctx* ctx, int key, int64_t* value);
/* Status of the last failed call on ctx (ctx = NULL: of the last failed
 * spk_spar_sink_multi, which owns its contexts): category (spk_status), class
 * (spk_error_kind) and message. Returns the category. */
int spk_last_error(const spk_ctx* ctx, int* category, int* kind, char* msg, size_t len);
/* Number of kernels this context has launched so far. */
int64_t spk_ctx_launch_count(const spk_ctx* ctx);

/* ---- end-to-end solvers ---------------------------------------------------- */

/* spar_sink_ot (uot = 0) / spar_sink_uot (uot = 1), solvers.hpp:159-167,
 * bodies solvers.cpp:314-378. a, b: n host weights. u, v (and log_u, log_v
 * when the log-domain path ran; may be NULL) receive n doubles each. */
int spk_spar_sink(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b,
                  const spk_solver_cfg* cfg, double s, uint64_t seed, const spk_sketch_opts* opts,
                  int uot, double* u, double* v, double* log_u, double* log_v, spk_report* rep);

/* Dense Sinkhorn: sinkhorn_ot / sinkhorn_uot on a KernelMatrix
 * (solvers.hpp:137-147). Dense form uploads K; coordinate form recomputes
 * K on the fly every iteration (config 5 comparator). The objective is
 * computed when a cost is available (dense C or coordinates). */
int spk_sinkhorn(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b,
                 const spk_solver_cfg* cfg, int uot, double* u, double* v, double* log_u,
                 double* log_v, spk_report* rep);

/* ---- device-resident sketch ------------------------------------------------ */

/* Plan (kind) -> [theta] -> poisson_sparsify on the device; builds CSR and
 * its CSC mirror. lambda/epsilon feed uot_probabilities (sparsify.cpp:93-115).
 * a and b are kept on the device for later solves. */
int spk_sketch_build(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b,
                     int plan_kind, double lambda, double epsilon, double s, uint64_t seed,
                     const spk_sketch_opts* opts, spk_sketch** out);
/* spk_sketch_build for `count` measure pairs on ONE kernel (pairwise_wfr's
 * frame pairs, harness.cpp:349-406): a and b are count x n row-major, seeds
 * count values; the kernel's coordinates, screen copies and support
 * threshold are prepared once. out: count sketches (all or none on error). */
int spk_sketch_build_batch(spk_ctx* ctx, const spk_kernel_desc* kd, int count, const double* a, const double* b,
                           int plan_kind, double lambda, double epsilon, double s, const uint64_t* seeds,
                           const spk_sketch_opts* opts, spk_sketch** out);
/* Upload a host CSR (SparseKernel layout, sparsify.hpp:57-71). */
int spk_sketch_from_csr(spk_ctx* ctx, int64_t n, const int64_t* row_ptr, const uint32_t* col_idx,
                        const double* values, int value_type, spk_sketch** out);
void spk_sketch_free(spk_sketch* sk);
int spk_sketch_info(const spk_sketch* sk, int64_t* n, int64_t* nnz, int64_t* kernel_nnz,
                    int32_t* factorized_plan, double* kernel_mean);
/* The sampling plan the sketch was drawn from: kind, factorized storage,
 * grid normaliser 1/total (masked_grid_plan, sparsify.cpp:65-67), UOT kernel
 * exponent eps/(2 lambda + eps) and theta. */
int spk_sketch_plan(const spk_sketch* sk, int32_t* plan_kind, int32_t* factorized, double* inv, double* g_k,
                    double* theta);
/* Copy CSR (row_ptr n+1, col_idx nnz, values nnz as fp64) / CSC to host. */
int spk_sketch_copy_csr(spk_sketch* sk, int64_t* row_ptr, uint32_t* col_idx, double* values);
int spk_sketch_copy_csc(spk_sketch* sk, int64_t* col_ptr, uint32_t* row_idx, double* values);
/* y = K~ x (transpose = 0) or K~' x (transpose = 1); host vectors of n. */
int spk_sketch_spmv(spk_sketch* sk, const double* x, double* y, int transpose);
/* Sinkhorn loop on the sketch. a/b NULL = the weights given at build. u, v,
 * log_u, log_v may be NULL (results stay on the device for readout). */
int spk_sketch_solve(spk_ctx* ctx, spk_sketch* sk, const double* a, const double* b,
                     const spk_solver_cfg* cfg, int uot, double* u, double* v, double* log_u,
                     double* log_v, spk_report* rep);
/* sinkhorn_uot / sinkhorn_ot<SparseKernel> on `count` independent sketches
 * (solvers.hpp:209-232; pairwise_wfr's per-pair solves, harness.cpp:349-406)
 * with the weights given at build. Log domain (cfg->stabilize) sketches small
 * enough for one CTA's shared memory run together, one CTA per sketch;
 * otherwise one after another. reps: `count` reports (may be NULL). Results
 * stay on each sketch for spk_sketch_readout / spk_sketch_scalings.
 * item_error NULL: on failure the status is that of the lowest failing item
 * and the message names it. item_error non-NULL (`count` entries): each
 * item's outcome is recorded there (0, or the SPK_E_* class of its failure:
 * ZeroDenominator, DegenerateSketchError, ...) and the call succeeds unless
 * the device faults -- pairwise_wfr's per-pair NaN (harness.cpp:395-401). */
int spk_sketch_solve_batch(spk_ctx* ctx, spk_sketch* const* sketches, int count, const spk_solver_cfg* cfg,
                           int uot, spk_report* reps, int32_t* item_error);
/* Scalings of the LAST solve on this sketch (n doubles each; any may be
 * NULL; log_u/log_v only after a log-domain solve) -- TransportPlan::u/v
 * (solvers.hpp:34-59). */
int spk_sketch_scalings(spk_sketch* sk, double* u, double* v, double* log_u, double* log_v);
/* Plan readout of the LAST solve on this sketch: marginals (may be NULL)
 * and the OT/UOT objective with costs from kd (dense C or coordinates). */
int spk_sketch_readout(spk_ctx* ctx, spk_sketch* sk, const spk_kernel_desc* kd, int uot,
                       double lambda, double epsilon, double* row_marginal, double* col_marginal,
                       double* objective, spk_report* rep);

/* Readout of a given plan T_ij = u_i K~_ij v_j (log domain: exp(lu + log K~ + lv))
 * over a host sketch (row_ptr != NULL: CSR of n rows) or over the kernel of kd
 * (dense K or coordinates; kd may also supply the costs). Replaces
 * TransportPlan::row_marginal / col_marginal (solvers.cpp:215-225),
 * ot_objective / uot_objective (:280-293) and marginal_residuals (:295-308).
 * a, b may be NULL when uot == 0 and no residuals are wanted. */
int spk_plan_readout(spk_ctx* ctx, const spk_kernel_desc* kd, int64_t n, const int64_t* row_ptr,
                     const uint32_t* col_idx, const double* values, const double* u, const double* v,
                     const double* log_u, const double* log_v, int log_domain, const double* a,
                     const double* b, int uot, double lambda, double epsilon, double* row_marginal,
                     double* col_marginal, double* objective, double* residual_row, double* residual_col);

/* ---- row/column-sharded Spar-Sink (one process per GPU) ----------------------
 *
 * rank r of a world of W owns atoms [r*m, min(n, (r+1)*m)),
 * m = ceil(n / W) -- those ROWS of K~ (sampled locally with the reference's
 * per-row RNG streams, so the union over ranks is bit-identical to the
 * single-GPU sketch) and those COLUMNS (a CSC assembled once by an
 * all-to-all of the row slabs' entries). Each half-step is then local: the
 * rank updates its slab of u (or v) from the full gathered v (or u), and
 * one all-gather (the caller's collective, NCCL over NVLink) completes the
 * vector. A gathered vector holds W blocks of `stride` = m + SPK_SHARD_TAIL
 * doubles: the rank's slab followed by its tail (residual partial, mask
 * count, first failing index), so the stop decisions ride on the same
 * collective and every rank takes them identically on the device without a
 * host round trip. Replaces the loop of detail::scaling_loop /
 * log_scaling_loop (solvers.hpp:256-513) for a row/column-partitioned
 * SparseKernel; the caller-side driver is paper_2306_06581_b200/sharded.py.
 * Buffers named *_dev are device pointers on the context's device. */
#define SPK_SHARD_TAIL 8
typedef struct spk_shard spk_shard;

/* Plan stage 1: the support / grid-normaliser pass (masked_grid_plan,
 * sparsify.cpp:49-67) over this rank's rows. *needs_pass = 0 when the plan
 * is factorized (no pass; outputs untouched). row_sum_dev / row_nnz_dev:
 * slab-length device arrays. */
int spk_shard_plan_rows(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b,
                        int plan_kind, double lambda, double epsilon, int32_t world, int32_t rank,
                        double* row_sum_dev, int64_t* row_nnz_dev, int32_t* needs_pass);
/* Plan stage 2 + poisson_sparsify of this rank's rows. row_sum_all_dev /
 * row_nnz_all_dev: the n per-row values of stage 1 gathered in rank order
 * (NULL when no pass is needed); the normaliser is their fixed-order total,
 * bit-identical to the single-GPU plan. kd must be the coordinate form. */
int spk_shard_create(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b,
                     int plan_kind, double lambda, double epsilon, double s, uint64_t seed,
                     const spk_sketch_opts* opts, int32_t world, int32_t rank,
                     const double* row_sum_all_dev, const int64_t* row_nnz_all_dev, spk_shard** out);
void spk_shard_free(spk_shard* sh);
/* Geometry and sizes: n, slab width m, gathered block stride, this rank's
 * slab [lo, hi), nnz of its row slab and (after import) of its column slab,
 * value bytes (4 or 8), its share of kernel_mean, kernel support, plan flag. */
int spk_shard_info(const spk_shard* sh, int64_t* n, int64_t* m, int64_t* stride, int64_t* lo, int64_t* hi,
                   int64_t* row_nnz, int64_t* col_nnz, int32_t* value_bytes, double* kernel_mean_part,
                   int64_t* kernel_nnz, int32_t* factorized_plan);
/* Column exchange, send side: the row slab's entries grouped by column
 * (rows ascending inside a column). counts_dev: W*m int64 per-column counts
 * (block d = columns owned by rank d, zero-padded to m); rows_dev: row_nnz
 * uint32 GLOBAL row indices; vals_dev: row_nnz values (value_bytes each);
 * send_sizes: W host int64 entry totals per destination. */
int spk_shard_export(spk_shard* sh, int64_t* counts_dev, uint32_t* rows_dev, void* vals_dev, int64_t* send_sizes);
/* Receive side: recv_counts_dev = W*m int64 (source-major), entries from
 * sources 0..W-1 concatenated in order (`total` of them). Builds the column
 * slab's CSC with rows ascending inside each column (spmv_t order). */
int spk_shard_import(spk_shard* sh, const int64_t* recv_counts_dev, const uint32_t* recv_rows_dev,
                     const void* recv_vals_dev, int64_t total);
/* Structural coverage of this rank's rows and columns (kernel_coverage,
 * solvers.cpp:138-163): empty counts of its slab. */
int spk_shard_coverage(spk_shard* sh, int64_t* empty_rows, int64_t* empty_cols);
/* Start a loop (sinkhorn_ot/uot checks, solvers.hpp:209-232, on the
 * weights given at create): totals of the coverage counts over all ranks
 * and the policy. Writes this rank's block (and tail) of u0_dev / v0_dev
 * (gathered-layout buffers); the caller all-gathers v0 before iteration 1. */
int spk_shard_begin(spk_shard* sh, const spk_solver_cfg* cfg, int uot, int policy, int64_t empty_rows_total,
                    int64_t empty_cols_total, double* u0_dev, double* v0_dev);
/* One half-step of iteration t >= 1. half 0: u-slab from x_dev = gathered
 * v of t-1 into out_dev (own block of gathered u of t), old_dev = gathered
 * u of t-1. half 1: v-slab from x_dev = gathered u of t, old_dev = gathered
 * v of t-1, out_dev = gathered v of t. First applies the decision of the
 * previous half (its tails in x_dev); no-op once the loop has stopped. */
int spk_shard_half(spk_shard* sh, int half, int64_t t, const double* x_dev, const double* old_dev, double* out_dev);
/* Decision on the v-half of iteration t_last (its gathered vector) after
 * the caller's last iteration. */
int spk_shard_finish(spk_shard* sh, int64_t t_last, const double* v_last_dev);
/* Loop state (synchronises): iterations, converged, diverged, masked
 * counts into rep; *stopped; *final_parity = which of the two ping-pong
 * buffers holds the result. Returns the reference's error status
 * (ZeroDenominator / DegenerateSketchError) when the loop raised. */
int spk_shard_status(spk_shard* sh, spk_report* rep, int32_t* stopped, int32_t* final_parity);
/* Readout partials of this rank (for_each_entry over its row slab, column
 * marginals over its column slab): out[0..7] = residual_row, residual_col,
 * <T,C>, H(T), KL row term, KL column term, first row with mass on an
 * infinite cost + 1 (0 = none), first atom with KL mass off support + 1. */
int spk_shard_readout(spk_shard* sh, const double* u_dev, const double* v_dev, int log_domain, int uot,
                      int want_objective, double* out);

/* ---- multi-GPU through the library: communicators + the sharded driver ------
 *
 * The collectives of the sharded solve above, owned by the library so a C /
 * C++ caller reaches config 4 on several GPUs (SURVEY §8(b) C-ABI row,
 * §8(e)). NCCL is loaded at run time (the copy already in the process, else
 * $SPK_NCCL_LIB, else libnccl.so.2). One rank per process (spk_comm_init with
 * an id made by spk_comm_unique_id on one rank and shared out of band), or
 * one process driving several GPUs (spk_comm_init_all / spk_spar_sink_multi).
 * An emulated communicator (threads of one process sharing one GPU,
 * host-synchronised copies) exercises the same driver in tests. */
typedef struct spk_comm spk_comm;
typedef struct spk_comm_group spk_comm_group;
int spk_comm_unique_id(unsigned char id[128]);
/* Rank `rank` of `world` on ctx's device (ncclCommInitRank). */
int spk_comm_init(spk_ctx* ctx, const unsigned char id[128], int world, int rank, spk_comm** out);
/* One process, ndev devices: ctxs[r] must be a context on devices[r]; comms[r] receives rank r. */
int spk_comm_init_all(const int* devices, int ndev, spk_ctx** ctxs, spk_comm** comms);
/* Emulated ranks: a host group of `world` threads; rank r's communicator on ctx. */
int spk_comm_group_create(int world, spk_comm_group** out);
void spk_comm_group_destroy(spk_comm_group* group);
int spk_comm_init_emulated(spk_ctx* ctx, spk_comm_group* group, int rank, spk_comm** out);
void spk_comm_destroy(spk_comm* comm);
int spk_comm_info(const spk_comm* comm, int* world, int* rank, int* nccl_backed);

/* This rank's share of a row/column-sharded sketch (build_sketch,
 * solvers.cpp:314-335, over the communicator's ranks: plan row sums
 * gathered in rank order, local sampling, the column all-to-all, coverage
 * totals). Every rank passes the same inputs. kd: coordinate form. */
typedef struct spk_sharded spk_sharded;
int spk_sharded_build(spk_comm* comm, const spk_kernel_desc* kd, const double* a, const double* b, int plan_kind,
                      double lambda, double epsilon, double s, uint64_t seed, const spk_sketch_opts* opts,
                      spk_sharded** out);
/* sinkhorn_ot / sinkhorn_uot<SparseKernel> (solvers.hpp:209-232) on the
 * sharded sketch, then the objective (rank-order sums). Every rank gets the
 * full u, v (and log_u, log_v after a log-domain solve; any may be NULL) and
 * the same report. With NCCL the iteration loop (per iteration: 2 half
 * kernels + 2 all-gathers) runs as one captured CUDA graph, replayed by later
 * solves with the same configuration: no host work per half-step. */
int spk_sharded_solve(spk_sharded* sh, const spk_solver_cfg* cfg, int uot, double* u, double* v, double* log_u,
                      double* log_v, spk_report* rep);
/* n, total sketch entries, kernel support, this rank's slab [lo, hi), and
 * the kernel launches inside the captured loop graph (0 if none). */
int spk_sharded_info(const spk_sharded* sh, int64_t* n, int64_t* nnz, int64_t* kernel_nnz, int64_t* lo, int64_t* hi,
                     int64_t* captured_launches);
void spk_sharded_free(spk_sharded* sh);
/* spar_sink_ot / spar_sink_uot (solvers.cpp:339-378) over the
 * communicator's ranks: build + solve + free. */
int spk_spar_sink_sharded(spk_comm* comm, const spk_kernel_desc* kd, const double* a, const double* b,
                          const spk_solver_cfg* cfg, double s, uint64_t seed, const spk_sketch_opts* opts, int uot,
                          double* u, double* v, double* log_u, double* log_v, spk_report* rep);
/* The same from ONE host thread over `ndev` GPUs of this process: contexts,
 * NCCL communicators (ncclCommInitAll) and one driver thread per GPU are
 * created and torn down inside. On failure spk_last_error(NULL, ...) reports
 * the failing rank's error. */
int spk_spar_sink_multi(const int* devices, int ndev, const spk_kernel_desc* kd, const double* a, const double* b,
                        const spk_solver_cfg* cfg, double s, uint64_t seed, const spk_sketch_opts* opts, int uot,
                        double* u, double* v, double* log_u, double* log_v, spk_report* rep);

/* ---- barycenters --------------------------------------------
 * BarycenterResult (barycenter.hpp:20-26) without the weights (written to q). */
typedef struct {
  int64_t iterations;
  int32_t converged;
  int32_t diverged;
  int64_t masked_atoms;
  double wall_time_s;
} spk_ibp_report;

/* ibp<SparseKernel> (barycenter.hpp:48-206) on m device sketches of one
 * dimension n: b = m x n host weights (row-major), w = m barycenter weights,
 * policy = spk_empty_policy. q receives the n barycenter weights. */
int spk_ibp(spk_ctx* ctx, spk_sketch* const* sketches, int32_t m, const double* b, const double* w, double delta,
            int64_t max_iter, int32_t policy, double* q, spk_ibp_report* rep);
/* spar_ibp (barycenter.cpp:8-40): sketch each kernel kds[k] with the
 * column-constant plan and seed mix_seed(seed, k), then ibp (Mask policy;
 * strict: orphan check + Error policy). */
int spk_spar_ibp(spk_ctx* ctx, const spk_kernel_desc* kds, int32_t m, const double* b, const double* w, double delta,
                 int64_t max_iter, double s, uint64_t seed, int32_t strict, int32_t value_type, double* q,
                 spk_ibp_report* rep);

/* ---- helpers exposed for parity tests --------------------------------------- */

/* SamplingPlan::prob(i, j) (sparsify.hpp:28-34) of the plan that
 * spk_sketch_build would use, for m query pairs. */
int spk_plan_probs(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b,
                   int plan_kind, double lambda, double epsilon, double theta, int64_t m,
                   const int64_t* qi, const int64_t* qj, double* probs, int32_t* factorized);

/* kernel_from_cost (geometry.cpp:83-102) on `count` host cost entries:
 * K = isinf(C) ? 0 : exp(-C/eps); *nnz = #(K > 0). */
int spk_kernel_from_cost(spk_ctx* ctx, const double* C, int64_t count, double epsilon, double* K, int64_t* nnz);

/* Cost and Gibbs kernel entries from coordinates (pairwise_cost +
 * kernel_from_cost) for m query pairs; c0 = max finite cost over all n^2
 * pairs when requested (NULL skips). */
int spk_cost_kernel(spk_ctx* ctx, const spk_kernel_desc* kd, int64_t m, const int64_t* qi,
                    const int64_t* qj, double* cost, double* kernel, double* c0);

#ifdef __cplusplus
}
#endif

#endif /* SPK_H_ */
