// spk_api.cu -- the C ABI (include/spk.h): context, error contract and the
// reference-facing entry points. Orchestration mirrors
// proj/src/solvers.cpp:314-378 (build_sketch + spar_sink_ot/uot) and
// include/sparsink/solvers.hpp:209-232 (sinkhorn_ot/uot). Host work is O(n):
// argument checks and the row/column weights that must be bit-identical to
// the reference; everything O(n^2) or O(nnz) runs on the device.
#include <cuda_runtime.h>

#include <chrono>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <new>
#include <string>

#include "internal.h"

namespace spk {

namespace {

const char* class_name(int kind) {
  switch (kind) {
    case SPK_E_NEGATIVE_WEIGHT: return "NegativeWeight";
    case SPK_E_LENGTH_MISMATCH: return "LengthMismatch";
    case SPK_E_NOT_NORMALIZED: return "NotNormalized";
    case SPK_E_ALL_BLACK: return "AllBlack";
    case SPK_E_EMPTY_OUTPUT: return "EmptyOutput";
    case SPK_E_DIMENSION_MISMATCH: return "DimensionMismatch";
    case SPK_E_NON_POSITIVE_ETA: return "NonPositiveEta";
    case SPK_E_NON_POSITIVE_EPSILON: return "NonPositiveEpsilon";
    case SPK_E_DEGENERATE_SUPPORT: return "DegenerateSupport";
    case SPK_E_ALL_ZERO_KERNEL: return "AllZeroKernel";
    case SPK_E_THETA_OUT_OF_RANGE: return "ThetaOutOfRange";
    case SPK_E_BUDGET_TOO_LARGE: return "BudgetTooLarge";
    case SPK_E_EMPTY_WINDOW: return "EmptyWindow";
    case SPK_E_INFINITE_COST_ON_SUPPORT: return "InfiniteCostOnSupport";
    case SPK_E_IO_ERROR: return "IoError";
    case SPK_E_ZERO_DENOMINATOR: return "ZeroDenominator";
    case SPK_E_BASELINE_FAILED: return "BaselineFailed";
    case SPK_E_DEGENERATE_SKETCH_ERROR: return "DegenerateSketchError";
    default: return nullptr;
  }
}

// errors.hpp:30-47: category of each class.
int category_of(int kind) {
  switch (kind) {
    case SPK_E_ZERO_DENOMINATOR:
    case SPK_E_BASELINE_FAILED: return SPK_STATUS_SOLVER;
    case SPK_E_DEGENERATE_SKETCH_ERROR: return SPK_STATUS_DEGENERATE_SKETCH;
    case SPK_E_DEVICE: return SPK_STATUS_DEVICE;
    default: return SPK_STATUS_INPUT;
  }
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

std::mutex g_proc_err_mu;
int g_proc_err_cat = 0, g_proc_err_kind = 0;
std::string g_proc_err_msg;

void init_report(spk_report* rep) {
  if (!rep) return;
  std::memset(rep, 0, sizeof *rep);
  rep->objective = std::numeric_limits<double>::quiet_NaN();
  rep->sketch_nnz = -1;
}

void check_cfg(const spk_solver_cfg* cfg) {
  if (!cfg) fail(SPK_E_LENGTH_MISMATCH, "null solver config");
  if (cfg->max_iter < 0) fail(SPK_E_LENGTH_MISMATCH, "max_iter must be >= 0");
}

void copy_scalings(spk_ctx* ctx, spk_sketch* sk, int64_t n, int log_domain, double* u, double* v, double* lu,
                   double* lv) {
  if (u) download(ctx, u, sk->u, sizeof(double) * n);
  if (v) download(ctx, v, sk->v, sizeof(double) * n);
  if (log_domain) {
    if (lu) download(ctx, lu, sk->lu, sizeof(double) * n);
    if (lv) download(ctx, lv, sk->lv, sizeof(double) * n);
  }
}

// Sinkhorn loop + report on a device sketch (the body of
// sinkhorn_ot/uot<SparseKernel>, solvers.hpp:209-232 + 256-513).
void solve_on_sketch(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, int uot, int policy, spk_report* rep) {
  const double f = solver_exponent(cfg, uot, sk->a_total, sk->b_total);
  LoopState st;
  st.n = sk->n;
  st.a = sk->a.as<double>();
  st.b = sk->b.as<double>();
  st.u = &sk->u;
  st.v = &sk->v;
  st.lu = &sk->lu;
  st.lv = &sk->lv;
  LoopOut lo;
  sk->last_valid = 0;
  run_sparse_loop(ctx, sk, cfg, f, policy, st, lo);
  sk->last_valid = 1;
  sk->last_log_domain = cfg.stabilize ? 1 : 0;
  sk->masked_rows = lo.masked_rows;
  sk->masked_cols = lo.masked_cols;
  // residuals from the plan marginals (solvers.hpp:380-389)
  ReadoutOut ro;
  Timer tr(ctx->stream);
  sparse_readout(ctx, sk, nullptr, sk->last_log_domain, st.a, st.b, false, uot, cfg.lambda, cfg.epsilon, nullptr,
                 nullptr, ro);
  const double t_read = tr.stop();
  if (rep) {
    rep->iterations = lo.iterations;
    rep->converged = lo.converged;
    rep->diverged = lo.diverged;
    rep->masked_rows = lo.masked_rows;
    rep->masked_cols = lo.masked_cols;
    rep->residual_row = ro.residual_row;
    rep->residual_col = ro.residual_col;
    rep->kernel_mean = sk->kernel_mean;
    rep->log_domain = sk->last_log_domain;
    rep->t_loop_s = lo.loop_s;
    rep->t_readout_s = t_read;
    rep->wall_time_s = lo.loop_s + t_read;
    rep->sketch_nnz = sk->nnz;
    rep->seed = sk->seed;
    rep->kernel_nnz = sk->kernel_nnz;
    rep->factorized_plan = sk->factorized_plan;
  }
}

void set_weights(spk_ctx* ctx, spk_sketch* sk, const double* a, const double* b) {
  upload(ctx, sk->a, a, sizeof(double) * sk->n);
  upload(ctx, sk->b, b, sizeof(double) * sk->n);
  sk->a_total = seq_total(a, sk->n);
  sk->b_total = seq_total(b, sk->n);
  sk->have_ab = true;
}

// build_sketch (solvers.cpp:314-335) into *sk; returns the plan timing.
void build_sketch(spk_ctx* ctx, DevKernel& dk, const double* a, const double* b, int plan_kind, double lambda,
                  double eps, double theta, double s, uint64_t seed, int value_type, spk_sketch* sk, double* t_plan,
                  double* t_sample) {
  PlanInfo plan;
  {
    NvtxRange r("spk:plan");
    Timer tp(ctx->stream);
    // UOT on a coordinate kernel: K^g_k enters every supported entry of the
    // grid normaliser as well. When a probe finds the support well filled,
    // K and K^g_k are evaluated once, before the plan pass, and both passes
    // stream them (config 2: plan 2.7 -> 1.5 ms including the evaluation).
    if (plan_kind == SPK_PLAN_UOT && !dk.dense && !ctx->force_two_pass && lambda > 0.0 && eps > 0.0 && !dk.cKg.p &&
        16.0 * (double)dk.n * (double)dk.n <= 8e9 && probe_support_fraction(ctx, dk) > 0.3)
      cache_uot_kernel(ctx, dk, eps / (2.0 * lambda + eps));
    build_plan(ctx, dk, a, b, plan_kind, lambda, eps, theta > 0.0 ? theta : 0.0, plan);
    *t_plan = tp.stop();
  }
  NvtxRange r("spk:sample");
  Timer ts(ctx->stream);
  // UOT on a coordinate kernel with a well-filled support: the tiled sampler
  // bounds K^g_k per entry with cos / log / exp2 and still takes the exact
  // exp / pow path for every candidate; evaluating K and K^g_k once for all
  // pairs and sampling from them is cheaper (config 2: 3.9 -> 1.8 ms). A
  // batch (spk_sketch_build_batch) has them already.
  if (plan_kind == SPK_PLAN_UOT && !dk.dense && !ctx->force_two_pass && !plan.factorized && lambda > 0.0 && eps > 0.0 &&
      (double)plan.kernel_nnz > 0.1 * (double)dk.n * (double)dk.n)
    cache_uot_kernel(ctx, dk, eps / (2.0 * lambda + eps));
  sample_sketch(ctx, dk, plan, s, seed, value_type, sk);
  *t_sample = ts.stop();
  set_weights(ctx, sk, a, b);
}

void strict_coverage(spk_ctx* ctx, spk_sketch* sk) {
  // solvers.cpp:325-333: first atom whose sketch row or column is empty
  std::vector<long long> rp(sk->n + 1), cp(sk->n + 1);
  download(ctx, rp.data(), sk->row_ptr, sizeof(long long) * (sk->n + 1));
  download(ctx, cp.data(), sk->col_ptr, sizeof(long long) * (sk->n + 1));
  for (int64_t i = 0; i < sk->n; ++i)
    if (rp[i + 1] == rp[i] || cp[i + 1] == cp[i])
      fail(SPK_E_DEGENERATE_SKETCH_ERROR,
           "sketch orphaned atom " + std::to_string(i) + "; raise s or theta, or use a different seed");
}

}  // namespace

// sinkhorn_ot / sinkhorn_uot argument checks (solvers.hpp:213-216, :226-228);
// returns the exponent f.
double solver_exponent(const spk_solver_cfg& cfg, int uot, double a_total, double b_total) {
  if (!uot) {
    if (std::abs(a_total - 1.0) > 1e-8 || std::abs(b_total - 1.0) > 1e-8)
      fail(SPK_E_NOT_NORMALIZED, "sinkhorn_ot requires simplex inputs");
    return 1.0;
  }
  if (!(cfg.lambda > 0) || !std::isfinite(cfg.lambda)) fail(SPK_E_ERROR, "sinkhorn_uot needs finite lambda > 0");
  return cfg.lambda / (cfg.lambda + cfg.epsilon);
}

void set_process_error(int category, int kind, const std::string& msg) {
  std::lock_guard<std::mutex> lk(g_proc_err_mu);
  g_proc_err_cat = category;
  g_proc_err_kind = kind;
  g_proc_err_msg = msg;
}

[[noreturn]] void fail(int kind, const std::string& text) {
  const char* cls = class_name(kind);
  throw Failure(category_of(kind), kind, cls ? std::string(cls) + ": " + text : text);
}

[[noreturn]] void fail_device(const char* what, cudaError_t e) {
  throw Failure(SPK_STATUS_DEVICE, SPK_E_DEVICE,
                std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ") in " + what);
}

thread_local cudaStream_t g_alloc_stream = nullptr;

void upload(spk_ctx* ctx, DBuf& dst, const void* src, size_t bytes) {
  dst.ensure(bytes ? bytes : 1);
  if (bytes) SPK_CUDA(cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
}

void download(spk_ctx* ctx, void* dst, const DBuf& src, size_t bytes) {
  if (!bytes) return;
  SPK_CUDA(cudaMemcpyAsync(dst, src.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  SPK_CUDA(cudaStreamSynchronize(ctx->stream));
}

double seq_total(const double* w, int64_t n) {
  double t = 0.0;
  for (int64_t i = 0; i < n; ++i) t += w[i];
  return t;
}

}  // namespace spk

using namespace spk;

extern "C" {

int spk_ctx_create(int device, spk_ctx** out) {
  if (!out) return SPK_STATUS_INPUT;
  *out = nullptr;
  auto ctx = std::make_unique<spk_ctx>();
  ctx->device = device;
  const int rc = guard(ctx.get(), [&] {
    int count = 0;
    SPK_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) fail_device("spk_ctx_create: no such device", cudaErrorInvalidDevice);
    SPK_CUDA(cudaSetDevice(device));
    SPK_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    int coop = 0;
    SPK_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    if (!coop) fail_device("device lacks cooperative launch", cudaErrorNotSupported);
    SPK_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    // device buffers come from the stream-ordered pool; keep freed memory in
    // it (a repeated solve then allocates nothing from the driver)
    cudaMemPool_t pool;
    SPK_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = ~0ull;
    SPK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    if (const char* e = std::getenv("SPK_STAGE_X")) ctx->stage_x = std::atoi(e) != 0;  // profiling
  });
  if (rc != SPK_OK) {
    std::fprintf(stderr, "spk_ctx_create: %s\n", ctx->err_msg.c_str());
    return rc;
  }
  *out = ctx.release();
  return SPK_OK;
}

void spk_ctx_destroy(spk_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  {
    AllocStreamScope scope(ctx->stream);
    ctx->scratch.release();
  }
  cudaStreamSynchronize(ctx->stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

int spk_ctx_set_stream(spk_ctx* ctx, void* stream) {
  if (!ctx) return SPK_STATUS_INPUT;
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  return SPK_OK;
}

void* spk_ctx_stream(spk_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int spk_ctx_set_option(spk_ctx* ctx, int key, int64_t value) {
  if (!ctx) return SPK_STATUS_INPUT;
  switch (key) {
    case SPK_OPT_DETERMINISTIC: ctx->deterministic = value ? 1 : 0; return SPK_OK;
    case SPK_OPT_LOOP_BLOCKS_PER_SM: ctx->loop_blocks_per_sm = (int)value; return SPK_OK;
    case 3: ctx->otf_fp32 = value ? 1 : 0; return SPK_OK;
    case 4: ctx->use_blocked = (int)std::max<int64_t>(0, std::min<int64_t>(value, 2)); return SPK_OK;
    case 5:  // multiple of 16 elements: every tile's TMA source stays 16-byte aligned
      ctx->blocked_max_w = (int)(std::max<int64_t>(16, std::min<int64_t>(value, 16384)) & ~int64_t(15));
      return SPK_OK;
    case 6: ctx->force_two_pass = value ? 1 : 0; return SPK_OK;
    case 9: ctx->blocked_cluster = value ? 1 : 0; return SPK_OK;
    case 10:
      if (value != 1 && value != 2 && value != 4) return SPK_STATUS_INPUT;
      ctx->batch_cluster = (int)value;
      return SPK_OK;
    case 11:
      if (value != 4 && value != 8) return SPK_STATUS_INPUT;
      ctx->batch_unroll = (int)value;
      return SPK_OK;
    case 12: ctx->small_loop = value ? 1 : 0; return SPK_OK;
    case 13:
      if (value != 1 && value != 2 && value != 4 && value != 8 && value != 16) return SPK_STATUS_INPUT;
      ctx->small_cluster = (int)value;
      return SPK_OK;
    case 14: ctx->small_max_nnz = std::max<int64_t>(0, value); return SPK_OK;
    case 15:
      if (value != 0 && value != 8 && value != 32) return SPK_STATUS_INPUT;
      ctx->row_lanes = (int)value;
      return SPK_OK;
    case 8: ctx->blocked_spread = value < 0 || value > 2 ? 1 : (int)value; return SPK_OK;
    case 7: ctx->blocked_split = (int)std::max<int64_t>(0, std::min<int64_t>(value, 2)); return SPK_OK;
    default: return SPK_STATUS_INPUT;
  }
}

int spk_ctx_get_option(const spk_ctx* ctx, int key, int64_t* value) {
  if (!ctx || !value) return SPK_STATUS_INPUT;
  switch (key) {
    case SPK_OPT_DETERMINISTIC: *value = ctx->deterministic; return SPK_OK;
    case SPK_OPT_LOOP_BLOCKS_PER_SM: *value = ctx->loop_blocks_per_sm; return SPK_OK;
    case 3: *value = ctx->otf_fp32; return SPK_OK;
    case 4: *value = ctx->use_blocked; return SPK_OK;
    case 5: *value = ctx->blocked_max_w; return SPK_OK;
    case 6: *value = ctx->force_two_pass; return SPK_OK;
    case 7: *value = ctx->blocked_split; return SPK_OK;
    case 8: *value = ctx->blocked_spread; return SPK_OK;
    case 9: *value = ctx->blocked_cluster; return SPK_OK;
    case 10: *value = ctx->batch_cluster; return SPK_OK;
    case 11: *value = ctx->batch_unroll; return SPK_OK;
    case 12: *value = ctx->small_loop; return SPK_OK;
    case 13: *value = ctx->small_cluster; return SPK_OK;
    case 14: *value = ctx->small_max_nnz; return SPK_OK;
    case 15: *value = ctx->row_lanes; return SPK_OK;
    default: return SPK_STATUS_INPUT;
  }
}

int spk_last_error(const spk_ctx* ctx, int* category, int* kind, char* msg, size_t len) {
  if (!ctx) {  // the last failure of a call that owns its contexts (spk_spar_sink_multi)
    std::lock_guard<std::mutex> lk(g_proc_err_mu);
    if (category) *category = g_proc_err_cat;
    if (kind) *kind = g_proc_err_kind;
    if (msg && len) std::snprintf(msg, len, "%s", g_proc_err_msg.c_str());
    return g_proc_err_cat;
  }
  if (category) *category = ctx->err_category;
  if (kind) *kind = ctx->err_kind;
  if (msg && len) std::snprintf(msg, len, "%s", ctx->err_msg.c_str());
  return ctx->err_category;
}

int64_t spk_ctx_launch_count(const spk_ctx* ctx) { return ctx ? ctx->launches : 0; }

int spk_spar_sink(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b,
                  const spk_solver_cfg* cfg, double s, uint64_t seed, const spk_sketch_opts* opts, int uot,
                  double* u, double* v, double* log_u, double* log_v, spk_report* rep) {
  if (!ctx) return SPK_STATUS_INPUT;
  init_report(rep);
  return guard(ctx, [&] {
    const double t0 = now_s();
    check_cfg(cfg);
    spk_sketch_opts o{};
    if (opts) o = *opts;
    DevKernel dk;
    make_dev_kernel(ctx, kd, cfg->epsilon, dk, /*need_cost=*/true);
    const int plan_kind = o.probs == SPK_PROBS_UNIFORM ? SPK_PLAN_UNIFORM : (uot ? SPK_PLAN_UOT : SPK_PLAN_OT);
    spk_sketch sk;
    sk.ctx = ctx;
    sk.device = ctx->device;
    double t_plan = 0, t_sample = 0;
    build_sketch(ctx, dk, a, b, plan_kind, cfg->lambda, cfg->epsilon, o.theta, s, seed, o.value_type, &sk, &t_plan,
                 &t_sample);
    if (o.strict) strict_coverage(ctx, &sk);
    solve_on_sketch(ctx, &sk, *cfg, uot, o.strict ? SPK_POLICY_ERROR : SPK_POLICY_MASK, rep);
    ReadoutOut ro;
    NvtxRange nr("spk:readout");
    Timer tr(ctx->stream);
    sparse_readout(ctx, &sk, &dk, sk.last_log_domain, sk.a.as<double>(), sk.b.as<double>(), true, uot, cfg->lambda,
                   cfg->epsilon, nullptr, nullptr, ro);
    const double t_obj = tr.stop();
    copy_scalings(ctx, &sk, sk.n, sk.last_log_domain, u, v, log_u, log_v);
    if (rep) {
      rep->objective = ro.objective;
      rep->sketch_nnz = sk.nnz;
      rep->seed = seed;
      rep->t_plan_s = t_plan;
      rep->t_sample_s = t_sample;
      rep->t_readout_s += t_obj;
      rep->wall_time_s = now_s() - t0;  // spar_sink_* report the total (solvers.cpp:353-355)
    }
  });
}

int spk_sinkhorn(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b,
                 const spk_solver_cfg* cfg, int uot, double* u, double* v, double* log_u, double* log_v,
                 spk_report* rep) {
  if (!ctx) return SPK_STATUS_INPUT;
  init_report(rep);
  return guard(ctx, [&] {
    check_cfg(cfg);
    if (!kd) fail(SPK_E_LENGTH_MISMATCH, "null kernel descriptor");
    const int64_t n = kd->n;
    const double f = solver_exponent(*cfg, uot, seq_total(a, n), seq_total(b, n));
    DevKernel dk;
    make_dev_kernel(ctx, kd, cfg->epsilon, dk, /*need_cost=*/true);
    if (!dk.dense) {  // coordinate form: kernel_from_cost's nnz_ratio is not needed by the loop
      dk.nnz_ratio = 1.0;
    }
    DBuf da, db, du, dv, dlu, dlv;
    upload(ctx, da, a, sizeof(double) * n);
    upload(ctx, db, b, sizeof(double) * n);
    LoopState st;
    st.n = n;
    st.a = da.as<double>();
    st.b = db.as<double>();
    st.u = &du;
    st.v = &dv;
    st.lu = &dlu;
    st.lv = &dlv;
    LoopOut lo;
    run_dense_loop(ctx, dk, *cfg, f, cfg->empty_policy, st, lo);
    const int log_domain = cfg->stabilize ? 1 : 0;
    ReadoutOut ro;
    Timer tr(ctx->stream);
    dense_readout(ctx, dk, log_domain, du, dv, dlu, dlv, st.a, st.b, dk.have_cost, uot, cfg->lambda, cfg->epsilon,
                  ro);
    const double t_read = tr.stop();
    if (u) download(ctx, u, du, sizeof(double) * n);
    if (v) download(ctx, v, dv, sizeof(double) * n);
    if (log_domain) {
      if (log_u) download(ctx, log_u, dlu, sizeof(double) * n);
      if (log_v) download(ctx, log_v, dlv, sizeof(double) * n);
    }
    if (rep) {
      rep->objective = ro.have_objective ? ro.objective : std::numeric_limits<double>::quiet_NaN();
      rep->iterations = lo.iterations;
      rep->converged = lo.converged;
      rep->diverged = lo.diverged;
      rep->masked_rows = lo.masked_rows;
      rep->masked_cols = lo.masked_cols;
      rep->residual_row = ro.residual_row;
      rep->residual_col = ro.residual_col;
      rep->log_domain = log_domain;
      rep->t_loop_s = lo.loop_s;
      rep->t_readout_s = t_read;
      rep->wall_time_s = lo.loop_s + t_read;
      rep->sketch_nnz = -1;
    }
  });
}

int spk_sketch_build(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b, int plan_kind,
                     double lambda, double epsilon, double s, uint64_t seed, const spk_sketch_opts* opts,
                     spk_sketch** out) {
  if (!ctx || !out) return SPK_STATUS_INPUT;
  *out = nullptr;
  return guard(ctx, [&] {
    spk_sketch_opts o{};
    if (opts) o = *opts;
    DevKernel dk;
    make_dev_kernel(ctx, kd, epsilon, dk, /*need_cost=*/false);
    auto sk = std::make_unique<spk_sketch>();
    sk->ctx = ctx;
    sk->device = ctx->device;
    double tp = 0, ts = 0;
    build_sketch(ctx, dk, a, b, plan_kind, lambda, epsilon, o.theta, s, seed, o.value_type, sk.get(), &tp, &ts);
    if (o.strict) strict_coverage(ctx, sk.get());
    *out = sk.release();
  });
}

int spk_sketch_build_batch(spk_ctx* ctx, const spk_kernel_desc* kd, int count, const double* a, const double* b,
                           int plan_kind, double lambda, double epsilon, double s, const uint64_t* seeds,
                           const spk_sketch_opts* opts, spk_sketch** out) {
  if (!ctx || !out || (count > 0 && (!a || !b || !seeds))) return SPK_STATUS_INPUT;
  for (int k = 0; k < count; ++k) out[k] = nullptr;
  return guard(ctx, [&] {
    spk_sketch_opts o{};
    if (opts) o = *opts;
    DevKernel dk;  // coordinates, fp32 screen copies and the support threshold: once for the batch
    make_dev_kernel(ctx, kd, epsilon, dk, /*need_cost=*/false);
    const int64_t n = dk.n;
    // UOT plans: K^g_k (and K) are the same n x n matrices for every pair of the
    // batch -- evaluated once when they fit, streamed by every pair's passes
    if (plan_kind == SPK_PLAN_UOT && count >= 2 && lambda > 0.0 && epsilon > 0.0 && !ctx->force_two_pass)
      cache_uot_kernel(ctx, dk, epsilon / (2.0 * lambda + epsilon));
    std::vector<std::unique_ptr<spk_sketch>> made;
    WeightCache wcache;
    struct CacheScope {
      spk_ctx* c;
      ~CacheScope() { c->wcache = nullptr; }
    } scope{ctx};
    ctx->wcache = &wcache;
    for (int k = 0; k < count; ++k) {
      auto sk = std::make_unique<spk_sketch>();
      sk->ctx = ctx;
      sk->device = ctx->device;
      double tp = 0, ts = 0;
      build_sketch(ctx, dk, a + (int64_t)k * n, b + (int64_t)k * n, plan_kind, lambda, epsilon, o.theta, s, seeds[k],
                   o.value_type, sk.get(), &tp, &ts);
      if (o.strict) strict_coverage(ctx, sk.get());
      made.push_back(std::move(sk));
    }
    for (int k = 0; k < count; ++k) out[k] = made[k].release();
  });
}

int spk_sketch_from_csr(spk_ctx* ctx, int64_t n, const int64_t* row_ptr, const uint32_t* col_idx,
                        const double* values, int value_type, spk_sketch** out) {
  if (!ctx || !out) return SPK_STATUS_INPUT;
  *out = nullptr;
  return guard(ctx, [&] {
    if (n <= 0) fail(SPK_E_LENGTH_MISMATCH, "sketch dimension must be positive");
    const int64_t nnz = row_ptr[n];
    auto sk = std::make_unique<spk_sketch>();
    sk->ctx = ctx;
    sk->device = ctx->device;
    sk->n = n;
    sk->nnz = nnz;
    sk->value_type = value_type;
    upload(ctx, sk->row_ptr, row_ptr, sizeof(int64_t) * (n + 1));
    upload(ctx, sk->col_idx, col_idx, sizeof(uint32_t) * nnz);
    if (value_type == SPK_VALUES_F32) {
      std::vector<float> f(nnz);
      for (int64_t k = 0; k < nnz; ++k) f[k] = (float)values[k];
      upload(ctx, sk->values, f.data(), sizeof(float) * nnz);
    } else {
      upload(ctx, sk->values, values, sizeof(double) * nnz);
    }
    SPK_CUDA(cudaStreamSynchronize(ctx->stream));
    build_csc(ctx, sk.get());
    sk->kernel_mean = sketch_kernel_mean(ctx, sk.get());
    *out = sk.release();
  });
}

void spk_sketch_free(spk_sketch* sk) {
  if (!sk) return;
  // the owning context (and its stream) may already be gone: only the device
  // id is used; once the device is idle the buffers go back to the pool
  cudaSetDevice(sk->device);
  cudaDeviceSynchronize();
  {
    AllocStreamScope scope(nullptr);
    delete sk;
  }
  (void)cudaGetLastError();
}

int spk_sketch_info(const spk_sketch* sk, int64_t* n, int64_t* nnz, int64_t* kernel_nnz, int32_t* factorized_plan,
                    double* kernel_mean) {
  if (!sk) return SPK_STATUS_INPUT;
  if (n) *n = sk->n;
  if (nnz) *nnz = sk->nnz;
  if (kernel_nnz) *kernel_nnz = sk->kernel_nnz;
  if (factorized_plan) *factorized_plan = sk->factorized_plan;
  if (kernel_mean) *kernel_mean = sk->kernel_mean;
  return SPK_OK;
}

int spk_sketch_plan(const spk_sketch* sk, int32_t* plan_kind, int32_t* factorized, double* inv, double* g_k,
                    double* theta) {
  if (!sk) return SPK_STATUS_INPUT;
  if (plan_kind) *plan_kind = sk->plan_kind;
  if (factorized) *factorized = sk->factorized_plan;
  if (inv) *inv = sk->plan_inv;
  if (g_k) *g_k = sk->plan_g_k;
  if (theta) *theta = sk->plan_theta;
  return SPK_OK;
}

static int copy_triplets(spk_sketch* sk, int csc, int64_t* ptr, uint32_t* idx, double* values) {
  return guard(sk->ctx, [&] {
    spk_ctx* ctx = sk->ctx;
    const DBuf& p = csc ? sk->col_ptr : sk->row_ptr;
    const DBuf& ix = csc ? sk->row_idx : sk->col_idx;
    const DBuf& vv = csc ? sk->values_t : sk->values;
    if (ptr) download(ctx, ptr, p, sizeof(int64_t) * (sk->n + 1));
    if (idx) download(ctx, idx, ix, sizeof(uint32_t) * sk->nnz);
    if (values) {
      if (sk->value_type == SPK_VALUES_F32) {
        std::vector<float> f(sk->nnz);
        download(ctx, f.data(), vv, sizeof(float) * sk->nnz);
        for (int64_t k = 0; k < sk->nnz; ++k) values[k] = f[k];
      } else {
        download(ctx, values, vv, sizeof(double) * sk->nnz);
      }
    }
  });
}

int spk_sketch_copy_csr(spk_sketch* sk, int64_t* row_ptr, uint32_t* col_idx, double* values) {
  if (!sk) return SPK_STATUS_INPUT;
  return copy_triplets(sk, 0, row_ptr, col_idx, values);
}

int spk_sketch_copy_csc(spk_sketch* sk, int64_t* col_ptr, uint32_t* row_idx, double* values) {
  if (!sk) return SPK_STATUS_INPUT;
  return copy_triplets(sk, 1, col_ptr, row_idx, values);
}

int spk_sketch_solve(spk_ctx* ctx, spk_sketch* sk, const double* a, const double* b, const spk_solver_cfg* cfg,
                     int uot, double* u, double* v, double* log_u, double* log_v, spk_report* rep) {
  if (!ctx || !sk) return SPK_STATUS_INPUT;
  init_report(rep);
  return guard(ctx, [&] {
    check_cfg(cfg);
    if (a || b) {
      if (!a || !b) fail(SPK_E_LENGTH_MISMATCH, "both marginals must be given");
      set_weights(ctx, sk, a, b);
    }
    if (!sk->have_ab) fail(SPK_E_LENGTH_MISMATCH, "sketch has no marginals; pass a and b");
    solve_on_sketch(ctx, sk, *cfg, uot, cfg->empty_policy, rep);
    copy_scalings(ctx, sk, sk->n, sk->last_log_domain, u, v, log_u, log_v);
  });
}

int spk_sketch_solve_batch(spk_ctx* ctx, spk_sketch* const* sks, int count, const spk_solver_cfg* cfg, int uot,
                           spk_report* reps, int32_t* item_error) {
  if (!ctx || (count > 0 && !sks)) return SPK_STATUS_INPUT;
  for (int k = 0; k < count; ++k) {
    init_report(reps ? reps + k : nullptr);
    if (item_error) item_error[k] = 0;
  }
  return guard(ctx, [&] {
    check_cfg(cfg);
    if (count < 0) fail(SPK_E_LENGTH_MISMATCH, "negative batch size");
    const int policy = cfg->empty_policy;
    std::vector<double> f(count);
    bool batched = cfg->stabilize && !ctx->deterministic;
    const int64_t nmax = batch_max_n(ctx);
    for (int k = 0; k < count; ++k) {
      spk_sketch* sk = sks[k];
      if (!sk) fail(SPK_E_LENGTH_MISMATCH, "null sketch in batch");
      if (!sk->have_ab) fail(SPK_E_LENGTH_MISMATCH, "sketch has no marginals; pass a and b at build");
      f[k] = solver_exponent(*cfg, uot, sk->a_total, sk->b_total);
      if (sk->n > nmax || sk->n_cols) batched = false;
    }
    // per-item outcome: with item_error the batch carries on past a failing
    // item (pairwise_wfr marks that pair NaN, harness.cpp:395-401); without it
    // the call fails with the lowest failing item
    int first_bad = -1;
    std::vector<std::string> pre_errs(count);
    std::vector<int> pre_kinds(count, 0);
    auto item_failed = [&](int k, int kind, const std::string& msg) {
      pre_kinds[k] = kind;
      pre_errs[k] = msg;
      sks[k]->last_valid = 0;
      if (item_error) item_error[k] = kind;
      if (first_bad < 0) first_bad = k;
    };
    if (!batched) {  // one solve at a time (linear domain, parity mode, or large sketches)
      for (int k = 0; k < count; ++k) {
        try {
          solve_on_sketch(ctx, sks[k], *cfg, uot, policy, reps ? reps + k : nullptr);
        } catch (const Failure& e) {
          if (!item_error || e.kind == SPK_E_DEVICE) throw;
          item_failed(k, e.kind, e.what());
        }
      }
      return;
    }
    // structural coverage and the loop's entry checks (solvers.hpp:411-414)
    std::vector<spk_sketch*> run;
    std::vector<int> run_k;
    std::vector<double> run_f;
    for (int k = 0; k < count; ++k) {
      spk_sketch* sk = sks[k];
      ensure_coverage(ctx, sk);
      int kind = 0;
      std::string msg;
      if ((sk->cov_empty_rows || sk->cov_empty_cols) && policy == SPK_POLICY_ERROR) {
        kind = SPK_E_ZERO_DENOMINATOR;
        msg = "kernel has empty rows or columns";
      }
      if (sk->cov_empty_rows == sk->n || sk->cov_empty_cols == sk->n) {
        kind = SPK_E_DEGENERATE_SKETCH_ERROR;
        msg = "kernel has no entries at all";
      }
      if (kind) {
        if (!item_error) fail(kind, "batch item " + std::to_string(k) + ": " + msg);
        item_failed(k, kind, msg);
        continue;
      }
      run.push_back(sk);
      run_k.push_back(k);
      run_f.push_back(f[k]);
    }
    std::vector<LoopOut> outs;
    std::vector<std::string> errs;
    std::vector<int> kinds;
    run_batch_log(ctx, run.data(), (int)run.size(), *cfg, run_f, policy, outs, errs, kinds);
    for (size_t q = 0; q < run.size(); ++q) {
      const int k = run_k[q];
      spk_sketch* sk = sks[k];
      const LoopOut& lo = outs[q];
      sk->last_valid = kinds[q] ? 0 : 1;
      sk->last_log_domain = 1;
      sk->masked_rows = lo.masked_rows;
      sk->masked_cols = lo.masked_cols;
      if (kinds[q]) {
        sk->last_valid = 0;
        pre_kinds[k] = kinds[q];
        pre_errs[k] = errs[q];
        if (item_error) item_error[k] = kinds[q];
        if (first_bad < 0 || k < first_bad) first_bad = k;
        continue;
      }
      ReadoutOut ro;  // residuals from the plan marginals (solvers.hpp:380-389)
      Timer tr(ctx->stream);
      sparse_readout(ctx, sk, nullptr, 1, sk->a.as<double>(), sk->b.as<double>(), false, uot, cfg->lambda,
                     cfg->epsilon, nullptr, nullptr, ro);
      const double t_read = tr.stop();
      if (reps) {
        spk_report* rep = reps + k;
        rep->iterations = lo.iterations;
        rep->converged = lo.converged;
        rep->diverged = 0;
        rep->masked_rows = lo.masked_rows;
        rep->masked_cols = lo.masked_cols;
        rep->residual_row = ro.residual_row;
        rep->residual_col = ro.residual_col;
        rep->kernel_mean = sk->kernel_mean;
        rep->log_domain = 1;
        rep->t_loop_s = lo.loop_s;
        rep->t_readout_s = t_read;
        rep->wall_time_s = lo.loop_s + t_read;
        rep->sketch_nnz = sk->nnz;
        rep->seed = sk->seed;
        rep->kernel_nnz = sk->kernel_nnz;
        rep->factorized_plan = sk->factorized_plan;
      }
    }
    if (first_bad >= 0 && !item_error)
      fail(pre_kinds[first_bad], "batch item " + std::to_string(first_bad) + ": " + pre_errs[first_bad]);
  });
}

int spk_sketch_scalings(spk_sketch* sk, double* u, double* v, double* log_u, double* log_v) {
  if (!sk) return SPK_STATUS_INPUT;
  return guard(sk->ctx, [&] {
    if (!sk->last_valid) fail(SPK_E_LENGTH_MISMATCH, "no solve has run on this sketch");
    copy_scalings(sk->ctx, sk, sk->n, sk->last_log_domain, u, v, log_u, log_v);
  });
}

int spk_sketch_readout(spk_ctx* ctx, spk_sketch* sk, const spk_kernel_desc* kd, int uot, double lambda,
                       double epsilon, double* row_marginal, double* col_marginal, double* objective,
                       spk_report* rep) {
  if (!ctx || !sk) return SPK_STATUS_INPUT;
  return guard(ctx, [&] {
    if (!sk->last_valid) fail(SPK_E_LENGTH_MISMATCH, "no solve has run on this sketch");
    std::unique_ptr<DevKernel> dk;
    if (kd) {
      dk = std::make_unique<DevKernel>();
      make_dev_kernel(ctx, kd, epsilon, *dk, /*need_cost=*/true);
    }
    ReadoutOut ro;
    Timer tr(ctx->stream);
    sparse_readout(ctx, sk, dk.get(), sk->last_log_domain, sk->a.as<double>(), sk->b.as<double>(),
                   objective != nullptr, uot, lambda, epsilon, row_marginal, col_marginal, ro);
    const double t = tr.stop();
    if (objective) *objective = ro.have_objective ? ro.objective : std::numeric_limits<double>::quiet_NaN();
    if (rep) {
      rep->residual_row = ro.residual_row;
      rep->residual_col = ro.residual_col;
      rep->objective = ro.have_objective ? ro.objective : std::numeric_limits<double>::quiet_NaN();
      rep->t_readout_s = t;
    }
  });
}

int spk_sketch_spmv(spk_sketch* sk, const double* x, double* y, int transpose) {
  if (!sk) return SPK_STATUS_INPUT;
  return guard(sk->ctx, [&] {
    sketch_product(sk->ctx, sk, x, y, transpose);
  });
}

int spk_plan_readout(spk_ctx* ctx, const spk_kernel_desc* kd, int64_t n, const int64_t* row_ptr,
                     const uint32_t* col_idx, const double* values, const double* u, const double* v,
                     const double* log_u, const double* log_v, int log_domain, const double* a, const double* b,
                     int uot, double lambda, double epsilon, double* row_marginal, double* col_marginal,
                     double* objective, double* residual_row, double* residual_col) {
  if (!ctx) return SPK_STATUS_INPUT;
  return guard(ctx, [&] {
    if (n <= 0) fail(SPK_E_LENGTH_MISMATCH, "plan dimension must be positive");
    if (log_domain ? (!log_u || !log_v) : (!u || !v)) fail(SPK_E_LENGTH_MISMATCH, "plan scalings missing");
    if (uot && (!a || !b)) fail(SPK_E_LENGTH_MISMATCH, "uot_objective needs both marginals");
    std::unique_ptr<DevKernel> dk;
    if (kd) {
      dk = std::make_unique<DevKernel>();
      make_dev_kernel(ctx, kd, epsilon, *dk, /*need_cost=*/true);
      if (dk->n != n) fail(SPK_E_LENGTH_MISMATCH, "kernel dimension != plan dimension");
    }
    std::vector<double> zeros;
    if (!a || !b) zeros.assign(n, 0.0);
    DBuf da, db;
    upload(ctx, da, a ? a : zeros.data(), sizeof(double) * n);
    upload(ctx, db, b ? b : zeros.data(), sizeof(double) * n);
    ReadoutOut ro;
    const bool want_obj = objective != nullptr;
    if (row_ptr) {
      spk_sketch sk;
      sk.ctx = ctx;
      sk.device = ctx->device;
      sk.n = n;
      sk.nnz = row_ptr[n];
      sk.value_type = SPK_VALUES_F64;
      upload(ctx, sk.row_ptr, row_ptr, sizeof(int64_t) * (n + 1));
      upload(ctx, sk.col_idx, col_idx, sizeof(uint32_t) * sk.nnz);
      upload(ctx, sk.values, values, sizeof(double) * sk.nnz);
      build_csc(ctx, &sk);
      if (log_domain) {
        upload(ctx, sk.lu, log_u, sizeof(double) * n);
        upload(ctx, sk.lv, log_v, sizeof(double) * n);
      } else {
        upload(ctx, sk.u, u, sizeof(double) * n);
        upload(ctx, sk.v, v, sizeof(double) * n);
      }
      sparse_readout(ctx, &sk, dk.get(), log_domain, da.as<double>(), db.as<double>(), want_obj, uot, lambda,
                     epsilon, row_marginal, col_marginal, ro);
    } else {
      if (!dk) fail(SPK_E_LENGTH_MISMATCH, "spk_plan_readout needs a sketch or a kernel");
      DBuf du, dv, dlu, dlv;
      if (log_domain) {
        upload(ctx, dlu, log_u, sizeof(double) * n);
        upload(ctx, dlv, log_v, sizeof(double) * n);
      } else {
        upload(ctx, du, u, sizeof(double) * n);
        upload(ctx, dv, v, sizeof(double) * n);
      }
      dense_readout(ctx, *dk, log_domain, du, dv, dlu, dlv, da.as<double>(), db.as<double>(), want_obj, uot, lambda,
                    epsilon, ro, row_marginal, col_marginal);
    }
    if (objective) *objective = ro.have_objective ? ro.objective : std::numeric_limits<double>::quiet_NaN();
    if (residual_row) *residual_row = ro.residual_row;
    if (residual_col) *residual_col = ro.residual_col;
  });
}

int spk_plan_probs(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b, int plan_kind,
                   double lambda, double epsilon, double theta, int64_t m, const int64_t* qi, const int64_t* qj,
                   double* probs, int32_t* factorized) {
  if (!ctx) return SPK_STATUS_INPUT;
  return guard(ctx, [&] {
    DevKernel dk;
    make_dev_kernel(ctx, kd, epsilon, dk, false);
    PlanInfo plan;
    build_plan(ctx, dk, a, b, plan_kind, lambda, epsilon, theta, plan);
    if (factorized) *factorized = plan.factorized ? 1 : 0;
    if (m > 0) plan_probs_query(ctx, dk, plan, m, qi, qj, probs);
  });
}

int spk_kernel_from_cost(spk_ctx* ctx, const double* C, int64_t count, double epsilon, double* K, int64_t* nnz) {
  if (!ctx) return SPK_STATUS_INPUT;
  return guard(ctx, [&] { kernel_from_cost_dev(ctx, C, count, epsilon, K, nnz); });
}

int spk_cost_kernel(spk_ctx* ctx, const spk_kernel_desc* kd, int64_t m, const int64_t* qi, const int64_t* qj,
                    double* cost, double* kernel, double* c0) {
  if (!ctx) return SPK_STATUS_INPUT;
  return guard(ctx, [&] {
    if (!kd || kd->K) fail(SPK_E_DIMENSION_MISMATCH, "spk_cost_kernel needs the coordinate form");
    DevKernel dk;
    make_dev_kernel(ctx, kd, kd->kernel_epsilon, dk, true);
    if (c0) *c0 = dk.scale;
    if (m > 0) cost_kernel_query(ctx, dk, m, qi, qj, cost, kernel);
  });
}

}  // extern "C"
