// internal.h -- host-side structures shared by the CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/spk.h"

namespace spk {

// An error carrying the reference's exception class and category; thrown
// inside the library and converted to a status at the C ABI boundary.
struct Failure : std::runtime_error {
  int category;
  int kind;
  Failure(int cat, int k, const std::string& msg) : std::runtime_error(msg), category(cat), kind(k) {}
};

[[noreturn]] void fail(int kind, const std::string& text);  // maps kind -> category, prefixes class
// error record of calls that own their contexts (spk_last_error(NULL, ...))
void set_process_error(int category, int kind, const std::string& msg);
[[noreturn]] void fail_device(const char* what, cudaError_t e);

#define SPK_CUDA(x)                                  \
  do {                                               \
    cudaError_t e_ = (x);                            \
    if (e_ != cudaSuccess) ::spk::fail_device(#x, e_); \
  } while (0)

// Stream that device buffers are allocated / freed on: the context stream of
// the C ABI call in progress (set by guard() and the free functions).
// Buffers come from the device's stream-ordered memory pool (kept, not
// returned to the driver: repeated solves allocate nothing new), and every
// use of a context's buffers is ordered on that same stream.
extern thread_local cudaStream_t g_alloc_stream;
struct AllocStreamScope {
  cudaStream_t prev;
  explicit AllocStreamScope(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
  ~AllocStreamScope() { g_alloc_stream = prev; }
};

// Device buffer with RAII.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  explicit DBuf(size_t b) { alloc(b); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t b) {
    release();
    bytes = b;
    if (b) SPK_CUDA(cudaMallocAsync(&p, b, g_alloc_stream));
  }
  void ensure(size_t b) { if (b > bytes) alloc(b); }
  void release() {
    if (p) cudaFreeAsync(p, g_alloc_stream);
    p = nullptr;
    bytes = 0;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Reusable device scratch of one Sinkhorn loop / readout (kept per sketch so
// repeated solves allocate nothing).
struct LoopWs {
  DBuf row_ne, col_ne, dyn_row, dyn_col, u2, v2, la, lb, absdiff, part, flag, status, scalar, xchg, pair, slices;
};
struct ReadWs {
  DBuf row_m, col_m, row_c, row_h, terms, flag, tmp, sums, bad;
};

// Slab x block layout of one half of a sketch (blocked.cu).
// Auto mode of the slab x block loop: from this n on the layout is tried (and kept unless its chunk padding
// exceeds 80%). Config 5's sketch (n = 5e4, 87 entries per row): 27.0k against 16.5k iterations/s for the CSR
// loop; config 2 (n = 1e4, 4.8x padding): 24.3k against 28.3k.
constexpr int64_t kBlockedAutoMinN = int64_t(1) << 15;

struct BlockedHalf {
  int P;        // CTAs (= Q row slabs x S column parts)
  int S;        // column parts per row slab (1, or 2 = pairs of CTAs split x)
  int B, Bh;    // column blocks in all, per part
  int W;        // columns per block (one staged x tile)
  int64_t n_out, n_in;
  int64_t split;  // S = 2: input atoms [0, split) go to column part 0, the rest to part 1 (S = 1: n_in)
  const int* slab_row0;    // [Q+1] global row starts
  const long long* off;    // [P*NW*(Bh+1)] entry offsets of (CTA, warp, block); [Bh] = stream end
  const uint32_t* packed;  // row_local << 16 | col_local, 4-chunk groups interleaved per lane
  const void* val;         // f32 or f64, same order
};
struct BlockedHost {
  BlockedHalf h{};
  DBuf slab_row0, off, packed, val;
  int max_rows = 0;
  int64_t padded = 0;  // entries after chunk padding
  std::vector<long long> cta_entries;  // padded entries per CTA (load-balance diagnostics)
};

}  // namespace spk

// Device-resident sketch: CSR plus its CSC mirror (rows ascending inside
// every column, so column sums run in the reference's spmv_t order).
struct spk_sketch {
  spk_ctx* ctx = nullptr;  // must outlive every call but spk_sketch_free
  int device = 0;
  int64_t n = 0;         // rows (all atoms, or this shard's row slab)
  int64_t n_cols = 0;    // columns when != n (row slab of a sharded sketch), else 0
  int64_t row_base = 0;  // global index of local row 0
  int64_t nnz = 0;
  int value_type = SPK_VALUES_F64;  // storage of values / values_t
  spk::DBuf row_ptr, col_idx, values;   // int64[n+1], u32[nnz], f64|f32[nnz]
  spk::DBuf col_ptr, row_idx, values_t; // CSC
  spk::DBuf log_values, log_values_t;   // lazily built log K~ (same dtype)
  spk::DBuf log_packed, log_packed_t;   // batched loop, fp32 sketches: u64 per entry = log K~ (fp64, 37-bit
                                        // mantissa) with the 16-bit column / row index in the low bits
  spk::DBuf a, b;                       // f64[n] weights given at build
  bool have_ab = false;
  double a_total = 0.0, b_total = 0.0;
  uint64_t seed = 0;
  int64_t kernel_nnz = 0;
  int factorized_plan = 0;
  double kernel_mean = 0.0;
  int plan_kind = SPK_PLAN_OT;
  double plan_inv = 1.0, plan_g_k = 0.0, plan_theta = 0.0;  // the sampling plan used
  // state of the last solve (device)
  spk::DBuf u, v, lu, lv;  // f64[n]
  int last_log_domain = 0;
  int last_valid = 0;
  int64_t masked_rows = 0, masked_cols = 0;
  // structural coverage (kernel_coverage) computed once per sketch
  spk::DBuf cov_row, cov_col;
  long long cov_empty_rows = -1, cov_empty_cols = -1;
  spk::LoopWs ws;
  spk::ReadWs rws;
  // fast-path layouts (built lazily by the first fast-mode solve)
  bool blocked_tried = false;
  int loop_solves = 0;  // sparse-loop runs on this sketch (a mid-size sketch earns its slab x block layout on reuse)
  int blocked_stages = 0;
  std::unique_ptr<spk::BlockedHost> blk_rows, blk_cols;
};

struct spk_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  int deterministic = 0;
  int loop_blocks_per_sm = 0;  // 0 = occupancy-derived
  int otf_fp32 = 1;            // dense on-the-fly comparator computes K in fp32
  int use_blocked = 2;         // fast sparse loop layout: 0 CSR/CSC, 1 slab x block, 2 auto (n >= kBlockedAutoMinN and chunk padding <= 80%)
  int blocked_max_w = 16384;   // cap on the shared tile width (tests force many blocks)
  int blocked_split = 0;       // column parts per row slab: 0 auto, 1, 2
  int stage_x = 1;             // grid loop: stage the gathered vector in shared memory when n <= 24576 (SPK_STAGE_X=0 disables)
  int blocked_spread = 1;      // slab x block layout: 1 = chunks by edge colouring (row and column bank classes), 2 = greedy column dealing, 0 = plain
  int blocked_cluster = 1;     // CTA pairs as 2-CTA clusters (DSMEM partial sums) when they all fit
  int batch_cluster = 2;       // batched log loop: CTAs (SMs) per sketch, 1 / 2 / 4
  int batch_unroll = 8;        // batched log loop: entry loads in flight per lane, 4 / 8
  int small_loop = 1;          // fast-mode loop on one cluster for small sketches (small.cu)
  int small_cluster = 16;      // its cluster size (largest that launches; 16 = non-portable)
  int64_t small_max_n = 14000;       // ... when both scaling vectors fit every CTA's shared memory
  int64_t small_max_nnz = 4000000;   // ... and the sketch is small enough that 16 SMs stream it faster
                                     //     than a grid barrier pair costs
  int force_two_pass = 0;      // sampler: skip the single-pass tiled path (testing)
  int row_lanes = 0;           // grid loop, fast mode: lanes per row, 0 auto (8 for short rows), 8, 32
  int64_t launches = 0;
  // last error
  int err_category = 0;
  int err_kind = 0;
  std::string err_msg;
  // scratch
  spk::DBuf scratch;
  // Large per-build temporaries (sort keys, permutations, sampler pools): kept
  // for the context's lifetime and grown on demand. Allocating and freeing
  // gigabytes of them per sketch made the stream-ordered pool map fresh memory
  // every other build (0.2-0.3 s stalls in build_csc / build_blocked).
  spk::DBuf tmp[16];
  // Batched UOT builds: a^g / b^g of the measures already seen in this batch
  // (config 3's 496 pairs use 32 frames; the host pow of 2 n weights per pair
  // was a fifth of the batch's sketch time). Set for the duration of
  // spk_sketch_build_batch only.
  struct WeightCache* wcache = nullptr;
};

struct WeightCache {
  struct Entry {
    const double* src;  // the caller's row (alive for the duration of the call)
    unsigned long long hash;
    double exponent;
    std::vector<double> w;
  };
  std::vector<Entry> entries;
};

namespace spk {
inline DBuf& tmp_buf(spk_ctx* ctx, int slot, size_t bytes) {
  ctx->tmp[slot].ensure(bytes);
  return ctx->tmp[slot];
}
}  // namespace spk

namespace spk {

void upload(spk_ctx* ctx, DBuf& dst, const void* src, size_t bytes);
void download(spk_ctx* ctx, void* dst, const DBuf& src, size_t bytes);

// NVTX range over a phase (plan / sample / loop / readout / ...): visible in
// nsys / ncu timelines; free when no tool is attached (NVTX v3, header-only).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  double stop() {
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e-3;
  }
  ~Timer() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

// Sequential host sum exactly as new_measure (measures.cpp:18-23).
double seq_total(const double* w, int64_t n);
// sinkhorn_ot / sinkhorn_uot argument checks; returns the exponent f.
double solver_exponent(const spk_solver_cfg& cfg, int uot, double a_total, double b_total);

// Runs f, converting library failures into the C ABI status and the
// context's last-error record.
template <class F>
int guard(spk_ctx* ctx, F&& f) {
  AllocStreamScope scope(ctx ? ctx->stream : g_alloc_stream);
  try {
    if (ctx) SPK_CUDA(cudaSetDevice(ctx->device));
    (void)cudaGetLastError();  // drop stale non-sticky errors from other callers
    f();
    if (ctx) {
      ctx->err_category = 0;
      ctx->err_kind = 0;
      ctx->err_msg.clear();
    }
    return SPK_OK;
  } catch (const Failure& e) {
    if (ctx) {
      ctx->err_category = e.category;
      ctx->err_kind = e.kind;
      ctx->err_msg = e.what();
    }
    return e.category;
  } catch (const std::bad_alloc&) {
    if (ctx) {
      ctx->err_category = SPK_STATUS_DEVICE;
      ctx->err_kind = SPK_E_DEVICE;
      ctx->err_msg = "host allocation failed";
    }
    return SPK_STATUS_DEVICE;
  } catch (const std::exception& e) {
    if (ctx) {
      ctx->err_category = SPK_STATUS_DEVICE;
      ctx->err_kind = SPK_E_DEVICE;
      ctx->err_msg = e.what();
    }
    return SPK_STATUS_DEVICE;
  }
}


// Kernel source on the device: dense K (+C) or coordinates.
struct DevKernel {
  int64_t n = 0;
  bool dense = false;
  DBuf K, C;       // dense form (n*n f64); C optional
  DBuf x, y;       // coordinate form (n*dim f64)
  int dim = 0, kind = 0;
  double eta = 0.0, scale = 1.0, eps = 1.0;
  double nnz_ratio = 1.0;  // dense form: given; coordinate form: computed
  bool have_cost = false;
  bool max_normalised = false;  // scale == c0 (every finite C_ij <= 1)
  double max_abs = 0.0;         // largest |coordinate| (enables the fp32 support screen)
  DBuf xf, yf, xn, yn;          // fp32 coordinates + squared norms (built on first use)
  DBuf ytr;                     // per sampler column tile: max |y_j|
  double d0 = 0.0;              // support threshold on d^2 (threshold_kernel), once per kernel
  bool have_d0 = false;
  // Batched UOT sketches on one coordinate kernel (config 3: 496 frame pairs on
  // one pixel grid): K and K^g_k are the same n x n matrices for every pair, so
  // they are evaluated once (exp, pow per entry) and every pair's plan and
  // sampling passes stream them instead (sampler.cu: *_cached_kernel).
  DBuf cK, cKg;
  double cache_g = -1.0;  // the exponent cKg was built for
};

// Fill dk.cK / dk.cKg for UOT plans with exponent g_k when n^2 entries fit the budget; false otherwise.
bool cache_uot_kernel(spk_ctx* ctx, DevKernel& dk, double g_k);
// Fraction of nonzero kernel entries among 4096 pseudo-random pairs (coordinate form).
double probe_support_fraction(spk_ctx* ctx, DevKernel& dk);

void make_dev_kernel(spk_ctx* ctx, const spk_kernel_desc* kd, double default_eps, DevKernel& dk,
                     bool need_cost);

// ---- sampler.cu ----
struct PlanInfo {
  int kind = SPK_PLAN_OT;
  bool factorized = true;
  double theta = 0.0;      // lazy theta (factorized) or folded (grid)
  int64_t kernel_nnz = 0;  // support size used by theta
  double inv = 1.0;        // grid normaliser 1/total
  double g_k = 0.0;        // UOT kernel exponent
  std::vector<double> row_w, col_w;  // ra/cb, pa/pb, or 1/n
  // plan-pass outputs kept on the device (grid plans): per-row support size
  // and unnormalised row mass, used to size the sampler's row slots
  DBuf d_row_nnz, d_row_sum;  // indexed by GLOBAL row
  mutable DBuf d_rw, d_cw;    // row_w / col_w on the device (uploaded once: the plan pass and the sampler share them)
  bool have_rows = false;
  bool zero_mass = false;
};

void build_plan(spk_ctx* ctx, DevKernel& dk, const double* a, const double* b, int plan_kind,
                double lambda, double eps, double theta, PlanInfo& plan);
// The three stages of build_plan, separable so row slabs of the n^2 pass can
// run on different GPUs: host O(n) weights (returns whether the support /
// normaliser pass is needed), the pass over rows [row0, row1) into local
// arrays, and the fixed-order totals over plan.d_row_* (all n rows).
bool plan_weights(spk_ctx* ctx, DevKernel& dk, const double* a, const double* b, int plan_kind, double lambda,
                  double eps, PlanInfo& plan);
void plan_pass_rows(spk_ctx* ctx, DevKernel& dk, const PlanInfo& plan, int64_t row0, int64_t row1,
                    long long* row_nnz, double* row_sum);
void plan_finish(spk_ctx* ctx, DevKernel& dk, bool need_pass, double theta, PlanInfo& plan);
// Samples rows [row0, row1) (default: all) of the plan into sk (a row slab
// with global column indices when sharded).
void sample_sketch(spk_ctx* ctx, DevKernel& dk, const PlanInfo& plan, double s, uint64_t seed,
                   int value_type, spk_sketch* sk, int64_t row0 = 0, int64_t row1 = -1);
void build_csc(spk_ctx* ctx, spk_sketch* sk);
void cost_kernel_query(spk_ctx* ctx, DevKernel& dk, int64_t m, const int64_t* qi, const int64_t* qj,
                       double* cost, double* kern);
void kernel_from_cost_dev(spk_ctx* ctx, const double* C_host, int64_t count, double eps, double* K_host,
                          int64_t* nnz);
void plan_probs_query(spk_ctx* ctx, DevKernel& dk, const PlanInfo& plan, int64_t m,
                      const int64_t* qi, const int64_t* qj, double* out);

// ---- loop.cu ----
struct LoopOut {
  int64_t iterations = 0;
  int converged = 0, diverged = 0;
  int64_t masked_rows = 0, masked_cols = 0;
  double loop_s = 0.0;
};
// Runs the scaling loop on a sketch (sparse) or dense kernel; results in
// sk->u/v (linear) or sk->lu/lv (log) style buffers passed in.
struct LoopState {
  int64_t n = 0;
  const double* a = nullptr;  // device
  const double* b = nullptr;
  DBuf *u = nullptr, *v = nullptr, *lu = nullptr, *lv = nullptr;
};
void run_sparse_loop(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent,
                     int policy, LoopState& st, LoopOut& out);
void ensure_coverage(spk_ctx* ctx, spk_sketch* sk);
void ensure_log_values(spk_ctx* ctx, spk_sketch* sk);
// shard.cu: half/finish launches since spk_shard_begin (selects the loop-state
// buffer); a replayed CUDA graph of the loop sets it as if issued
void shard_set_calls(spk_shard* sh, long long calls);
// small.cu: the loop on one cluster (scalings in shared memory); false = not applicable
bool run_cluster_loop(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy,
                      LoopState& st, LoopOut& out);
// batch.cu: one CTA per sketch, log domain, scalings in shared memory
int64_t batch_max_n(spk_ctx* ctx);
void run_batch_log(spk_ctx* ctx, spk_sketch* const* sks, int count, const spk_solver_cfg& cfg,
                   const std::vector<double>& exponents, int policy, std::vector<LoopOut>& outs,
                   std::vector<std::string>& errors, std::vector<int>& error_kinds);
bool run_blocked(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy,
                 LoopState& st, LoopOut& out);
void run_dense_loop(spk_ctx* ctx, DevKernel& dk, const spk_solver_cfg& cfg, double exponent,
                    int policy, LoopState& st, LoopOut& out);

// ---- readout.cu ----
struct ReadoutOut {
  double residual_row = 0.0, residual_col = 0.0;
  double objective = 0.0;
  bool have_objective = false;
};
// Plan marginals, residuals and objective over the sketch support
// (for_each_entry semantics, T > 0 only).
void sparse_readout(spk_ctx* ctx, spk_sketch* sk, DevKernel* dk, int log_domain, const double* a,
                    const double* b, bool want_objective, int uot, double lambda, double eps,
                    double* row_m_host, double* col_m_host, ReadoutOut& out);
void dense_readout(spk_ctx* ctx, DevKernel& dk, int log_domain, const DBuf& u, const DBuf& v,
                   const DBuf& lu, const DBuf& lv, const double* a, const double* b,
                   bool want_objective, int uot, double lambda, double eps, ReadoutOut& out,
                   double* row_m_host = nullptr, double* col_m_host = nullptr);
double sketch_kernel_mean(spk_ctx* ctx, spk_sketch* sk);
// spmv / spmv_t on the device sketch in the reference's summation order.
void sketch_product(spk_ctx* ctx, spk_sketch* sk, const double* x_host, double* y_host, int transpose);

}  // namespace spk
