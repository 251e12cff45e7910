// sharded.cu -- the multi-GPU Spar-Sink driver inside the library (SURVEY
// §8(e), C ABI spk_sharded_* / spk_spar_sink_sharded / spk_spar_sink_multi).
//
// Rank r of W owns atoms [r m, min(n, (r+1) m)), m = ceil(n / W), as ROWS of
// K~ (sampled with the reference's per-row RNG streams, poisson_sparsify,
// proj/src/sparsify.cpp:184-198: the union over ranks is the 1-GPU sketch bit
// for bit) and as COLUMNS (a CSC assembled once by an all-to-all of the row
// slabs' entries). Each half-step of detail::scaling_loop /
// log_scaling_loop (proj/include/sparsink/solvers.hpp:256-513) is then local
// to the rank (spk_shard_half: slab x block layout, CTA-pair clusters) and
// ONE all-gather completes the scaling vector; the stop / divergence / mask
// decisions ride in the tail behind every rank's slab, so all ranks take them
// on the device. With NCCL the whole iteration loop (2 half kernels + 2
// all-gathers per iteration, every iteration) is captured once into a CUDA
// graph and replayed per solve: no host work per half-step. The emulated
// communicator (threads sharing one GPU, host-synchronised copies) runs the
// same sequence uncaptured.
//
// The same steps as the Python driver paper_2306_06581_b200/sharded.py
// (which tests/test_multigpu_gloo.py runs over gloo).
#include <chrono>
#include <cmath>
#include <mutex>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "comm.h"
#include "internal.h"

using namespace spk;

struct spk_sharded {
  spk_comm* comm = nullptr;
  spk_ctx* ctx = nullptr;
  spk_shard* sh = nullptr;
  int64_t n = 0, m = 0, stride = 0, lo = 0, hi = 0;
  int64_t empty_rows = 0, empty_cols = 0, nnz = 0, kernel_nnz = 0;
  int factorized = 0;
  double kernel_mean = 0.0;
  uint64_t seed = 0;
  int strict = 0;
  DBuf U[2], V[2], part;
  // captured loop (NCCL): replayed while the loop parameters match
  cudaGraphExec_t graph = nullptr;
  int64_t g_iters = -1;
  spk_solver_cfg g_cfg{};
  int g_uot = -1, g_policy = -1;
  int64_t g_launches = 0;
  ~spk_sharded() {
    if (graph) cudaGraphExecDestroy(graph);
    if (sh) spk_shard_free(sh);
  }
};

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void check_rc(spk_ctx* ctx, int rc) {
  if (rc == SPK_OK) return;
  int cat = 0, kind = 0;
  char buf[1024];
  spk_last_error(ctx, &cat, &kind, buf, sizeof buf);
  throw Failure(cat ? cat : SPK_STATUS_DEVICE, kind ? kind : SPK_E_DEVICE, buf);
}

void slab(int64_t n, int world, int rank, int64_t& m, int64_t& lo, int64_t& hi) {
  m = (n + world - 1) / world;
  lo = std::min<int64_t>(n, (int64_t)rank * m);
  hi = std::min<int64_t>(n, lo + m);
}

bool same_cfg(const spk_solver_cfg& a, const spk_solver_cfg& b) {
  return a.epsilon == b.epsilon && (a.lambda == b.lambda || (std::isinf(a.lambda) && std::isinf(b.lambda))) &&
         a.delta == b.delta && a.max_iter == b.max_iter && a.stabilize == b.stabilize;
}

// build_sketch (solvers.cpp:314-335) over W ranks.
void build(spk_sharded* S, const spk_kernel_desc* kd, const double* a, const double* b, int plan_kind, double lambda,
           double eps, double s, uint64_t seed, const spk_sketch_opts* opts) {
  spk_comm* comm = S->comm;
  spk_ctx* ctx = S->ctx;
  const int W = comm->world, r = comm->rank;
  cudaStream_t st = ctx->stream;
  NvtxRange nr("spk:sharded_build");
  const int64_t n = kd->n;
  int64_t m, lo, hi;
  slab(n, W, r, m, lo, hi);
  S->n = n;
  S->m = m;
  S->lo = lo;
  S->hi = hi;
  S->seed = seed;
  S->strict = opts && opts->strict;
  // 1. plan: this rank's support / normaliser rows, gathered in rank order
  DBuf rs(sizeof(double) * std::max<int64_t>(m, 1)), rn(sizeof(int64_t) * std::max<int64_t>(m, 1));
  int32_t need = 0;
  check_rc(ctx, spk_shard_plan_rows(ctx, kd, a, b, plan_kind, lambda, eps, W, r, rs.as<double>(), rn.as<int64_t>(),
                                    &need));
  DBuf rs_all, rn_all;
  if (need) {
    rs_all.alloc(sizeof(double) * W * m);
    rn_all.alloc(sizeof(int64_t) * W * m);
    SPK_CUDA(cudaMemcpyAsync(rs_all.as<double>() + r * m, rs.p, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
    SPK_CUDA(cudaMemcpyAsync(rn_all.as<int64_t>() + r * m, rn.p, sizeof(int64_t) * m, cudaMemcpyDeviceToDevice, st));
    comm->all_gather(rs_all.p, sizeof(double) * m, st);
    comm->all_gather(rn_all.p, sizeof(int64_t) * m, st);
  }
  // 2. sample this rank's rows
  check_rc(ctx, spk_shard_create(ctx, kd, a, b, plan_kind, lambda, eps, s, seed, opts, W, r,
                                 need ? rs_all.as<double>() : nullptr, need ? rn_all.as<int64_t>() : nullptr,
                                 &S->sh));
  rs_all.release();
  rn_all.release();
  int64_t nn, mm, stride, lo2, hi2, row_nnz, col_nnz, knnz;
  int32_t vbytes, fac;
  double km_part;
  check_rc(ctx, spk_shard_info(S->sh, &nn, &mm, &stride, &lo2, &hi2, &row_nnz, &col_nnz, &vbytes, &km_part, &knnz,
                               &fac));
  S->stride = stride;
  S->kernel_nnz = knnz;
  S->factorized = fac;
  // 3. column exchange: every rank's entries of my columns, sources in rank order
  DBuf counts(sizeof(int64_t) * W * m), rows(sizeof(uint32_t) * std::max<int64_t>(row_nnz, 1)),
      vals((size_t)vbytes * std::max<int64_t>(row_nnz, 1));
  std::vector<int64_t> send_sizes(W);
  check_rc(ctx, spk_shard_export(S->sh, counts.as<int64_t>(), rows.as<uint32_t>(), vals.p, send_sizes.data()));
  DBuf sizes_all(sizeof(int64_t) * W * W);
  SPK_CUDA(cudaMemcpyAsync(sizes_all.as<int64_t>() + r * W, send_sizes.data(), sizeof(int64_t) * W,
                           cudaMemcpyHostToDevice, st));
  comm->all_gather(sizes_all.p, sizeof(int64_t) * W, st);
  std::vector<int64_t> all(W * W);
  download(ctx, all.data(), sizes_all, sizeof(int64_t) * W * W);
  std::vector<int64_t> recv_sizes(W);
  int64_t total = 0;
  for (int src = 0; src < W; ++src) total += (recv_sizes[src] = all[src * W + r]);
  std::vector<int64_t> cb_send(W, (int64_t)sizeof(int64_t) * m), cb_recv(W, (int64_t)sizeof(int64_t) * m);
  DBuf recv_counts(sizeof(int64_t) * W * m);
  comm->all_to_all_v(counts.p, cb_send.data(), recv_counts.p, cb_recv.data(), st);
  DBuf recv_rows(sizeof(uint32_t) * std::max<int64_t>(total, 1)), recv_vals((size_t)vbytes * std::max<int64_t>(total, 1));
  std::vector<int64_t> sb(W), rb(W);
  for (int p = 0; p < W; ++p) {
    sb[p] = send_sizes[p] * 4;
    rb[p] = recv_sizes[p] * 4;
  }
  comm->all_to_all_v(rows.p, sb.data(), recv_rows.p, rb.data(), st);
  for (int p = 0; p < W; ++p) {
    sb[p] = send_sizes[p] * vbytes;
    rb[p] = recv_sizes[p] * vbytes;
  }
  comm->all_to_all_v(vals.p, sb.data(), recv_vals.p, rb.data(), st);
  counts.release();
  rows.release();
  vals.release();
  check_rc(ctx, spk_shard_import(S->sh, recv_counts.as<int64_t>(), recv_rows.as<uint32_t>(), recv_vals.p, total));
  recv_counts.release();
  recv_rows.release();
  recv_vals.release();
  // 4. coverage totals and sketch-wide scalars
  int64_t er, ec;
  check_rc(ctx, spk_shard_coverage(S->sh, &er, &ec));
  int64_t tot_h[3] = {er, ec, row_nnz};
  DBuf tot(sizeof tot_h);
  SPK_CUDA(cudaMemcpyAsync(tot.p, tot_h, sizeof tot_h, cudaMemcpyHostToDevice, st));
  comm->all_reduce_sum(tot.p, 3, CommType::I64, st);
  download(ctx, tot_h, tot, sizeof tot_h);
  S->empty_rows = tot_h[0];
  S->empty_cols = tot_h[1];
  S->nnz = tot_h[2];
  DBuf km(sizeof(double) * W);
  SPK_CUDA(cudaMemcpyAsync(km.as<double>() + r, &km_part, sizeof(double), cudaMemcpyHostToDevice, st));
  comm->all_gather(km.p, sizeof(double), st);
  std::vector<double> kmh(W);
  download(ctx, kmh.data(), km, sizeof(double) * W);
  S->kernel_mean = 0.0;
  for (double v : kmh) S->kernel_mean += v;  // rank order
  if (S->strict && (S->empty_rows || S->empty_cols))  // strict check (solvers.cpp:325-333)
    fail(SPK_E_DEGENERATE_SKETCH_ERROR, "sketch orphaned " + std::to_string(S->empty_rows) + " rows and " +
                                            std::to_string(S->empty_cols) +
                                            " columns; raise s or theta, or use a different seed");
  for (int k = 0; k < 2; ++k) {  // + 2 doubles: the last x tile's 16-byte-rounded TMA copy may read 8 bytes past
    S->U[k].alloc(sizeof(double) * (W * stride + 2));
    S->V[k].alloc(sizeof(double) * (W * stride + 2));
    SPK_CUDA(cudaMemsetAsync(S->U[k].p, 0, sizeof(double) * W * stride, st));
    SPK_CUDA(cudaMemsetAsync(S->V[k].p, 0, sizeof(double) * W * stride, st));
  }
  S->part.alloc(sizeof(double) * 8 * W);
  SPK_CUDA(cudaStreamSynchronize(st));
}

// Iterations 1..iters (two halves + two all-gathers each) and the final decision.
void loop_body(spk_sharded* S, int64_t iters) {
  spk_ctx* ctx = S->ctx;
  cudaStream_t st = ctx->stream;
  const size_t chunk = sizeof(double) * S->stride;
  double* U[2] = {S->U[0].as<double>(), S->U[1].as<double>()};
  double* V[2] = {S->V[0].as<double>(), S->V[1].as<double>()};
  int64_t t = 0;
  for (t = 1; t <= iters; ++t) {
    check_rc(ctx, spk_shard_half(S->sh, 0, t, V[(t - 1) & 1], U[(t - 1) & 1], U[t & 1]));
    S->comm->all_gather(U[t & 1], chunk, st);
    check_rc(ctx, spk_shard_half(S->sh, 1, t, U[t & 1], V[(t - 1) & 1], V[t & 1]));
    S->comm->all_gather(V[t & 1], chunk, st);
  }
  t = iters;
  check_rc(ctx, spk_shard_finish(S->sh, t, V[t & 1]));
}

void solve(spk_sharded* S, const spk_solver_cfg& cfg, int uot, double* u, double* v, double* lu, double* lv,
           spk_report* rep) {
  spk_comm* comm = S->comm;
  spk_ctx* ctx = S->ctx;
  cudaStream_t st = ctx->stream;
  const int W = comm->world, r = comm->rank;
  const int policy = S->strict ? SPK_POLICY_ERROR : SPK_POLICY_MASK;
  NvtxRange nr("spk:sharded_solve");
  const double t0 = now_s();
  Timer tm(st);
  check_rc(ctx, spk_shard_begin(S->sh, &cfg, uot, policy, S->empty_rows, S->empty_cols, S->U[0].as<double>(),
                                S->V[0].as<double>()));
  comm->all_gather(S->V[0].p, sizeof(double) * S->stride, st);
  const int64_t iters = cfg.max_iter;
  if (comm->capturable() && iters > 0) {
    const bool hit = S->graph && S->g_iters == iters && same_cfg(S->g_cfg, cfg) && S->g_uot == uot &&
                     S->g_policy == policy;
    if (!hit) {
      if (S->graph) {
        cudaGraphExecDestroy(S->graph);
        S->graph = nullptr;
      }
      const int64_t l0 = ctx->launches;
      cudaGraph_t g = nullptr;
      SPK_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      try {
        loop_body(S, iters);
      } catch (...) {
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      SPK_CUDA(cudaStreamEndCapture(st, &g));
      SPK_CUDA(cudaGraphInstantiate(&S->graph, g, 0));
      SPK_CUDA(cudaGraphDestroy(g));
      S->g_iters = iters;
      S->g_cfg = cfg;
      S->g_uot = uot;
      S->g_policy = policy;
      S->g_launches = ctx->launches - l0;
      ctx->launches = l0;
    }
    SPK_CUDA(cudaGraphLaunch(S->graph, st));
    ctx->launches += S->g_launches;
    shard_set_calls(S->sh, 2 * iters + 1);  // the captured halves + finish, as if issued now
  } else {
    loop_body(S, iters);
  }
  spk_report lr{};
  int32_t stopped = 0, par = 0;
  check_rc(ctx, spk_shard_status(S->sh, &lr, &stopped, &par));  // raises the loop's error like the reference
  const double loop_s = tm.stop();
  // readout partials, summed in rank order on every rank
  const bool log_domain = cfg.stabilize != 0;
  double part[8];
  check_rc(ctx, spk_shard_readout(S->sh, S->U[par].as<double>(), S->V[par].as<double>(), log_domain, uot, 1, part));
  SPK_CUDA(cudaMemcpyAsync(S->part.as<double>() + 8 * r, part, sizeof part, cudaMemcpyHostToDevice, st));
  comm->all_gather(S->part.p, sizeof part, st);
  std::vector<double> P(8 * W);
  download(ctx, P.data(), S->part, sizeof(double) * 8 * W);
  double sums[6] = {0, 0, 0, 0, 0, 0};
  int64_t inf_row = -1, kl_bad = -1;
  for (int q = 0; q < W; ++q) {
    for (int k = 0; k < 6; ++k) sums[k] += P[8 * q + k];
    if (P[8 * q + 6] > 0 && inf_row < 0) inf_row = (int64_t)P[8 * q + 6] - 1;
    if (P[8 * q + 7] > 0 && kl_bad < 0) kl_bad = (int64_t)P[8 * q + 7] - 1;
  }
  if (inf_row >= 0)
    fail(SPK_E_INFINITE_COST_ON_SUPPORT, "plan mass on a blocked entry (row " + std::to_string(inf_row) + ")");
  if (uot && kl_bad >= 0) fail(SPK_E_ERROR, "KL undefined: mass off support");
  const double lam = cfg.lambda, eps = cfg.epsilon;
  const double objective =
      uot ? (sums[2] + lam * sums[4] + lam * sums[5] - eps * sums[3]) : (sums[2] - eps * sums[3]);
  // scalings: strip the tails of the gathered vectors
  if (u || v || lu || lv) {
    std::vector<double> gu((size_t)W * S->stride), gv((size_t)W * S->stride);
    download(ctx, gu.data(), S->U[par], sizeof(double) * gu.size());
    download(ctx, gv.data(), S->V[par], sizeof(double) * gv.size());
    for (int64_t i = 0; i < S->n; ++i) {
      const int64_t blk = i / S->m, off = i - blk * S->m;
      const double x = gu[blk * S->stride + off], y = gv[blk * S->stride + off];
      if (log_domain) {
        if (lu) lu[i] = x;
        if (lv) lv[i] = y;
        if (u) u[i] = std::exp(x);
        if (v) v[i] = std::exp(y);
      } else {
        if (u) u[i] = x;
        if (v) v[i] = y;
      }
    }
  }
  if (rep) {
    *rep = lr;
    rep->objective = objective;
    rep->residual_row = sums[0];
    rep->residual_col = sums[1];
    rep->seed = S->seed;
    rep->kernel_mean = S->kernel_mean;
    rep->sketch_nnz = S->nnz;
    rep->kernel_nnz = S->kernel_nnz;
    rep->factorized_plan = S->factorized;
    rep->t_loop_s = loop_s;
    rep->wall_time_s = now_s() - t0;
  }
}

int plan_kind_of(const spk_sketch_opts* o, int uot) {
  if (o && o->probs == SPK_PROBS_UNIFORM) return SPK_PLAN_UNIFORM;
  return uot ? SPK_PLAN_UOT : SPK_PLAN_OT;
}

}  // namespace

extern "C" {

int spk_sharded_build(spk_comm* comm, const spk_kernel_desc* kd, const double* a, const double* b, int plan_kind,
                      double lambda, double epsilon, double s, uint64_t seed, const spk_sketch_opts* opts,
                      spk_sharded** out) {
  if (!comm || !comm->ctx || !kd || !a || !b || !out) return SPK_STATUS_INPUT;
  *out = nullptr;
  return guard(comm->ctx, [&] {
    auto S = std::make_unique<spk_sharded>();
    S->comm = comm;
    S->ctx = comm->ctx;
    build(S.get(), kd, a, b, plan_kind, lambda, epsilon, s, seed, opts);
    *out = S.release();
  });
}

int spk_sharded_solve(spk_sharded* S, const spk_solver_cfg* cfg, int uot, double* u, double* v, double* log_u,
                      double* log_v, spk_report* rep) {
  if (!S || !cfg) return SPK_STATUS_INPUT;
  return guard(S->ctx, [&] { solve(S, *cfg, uot, u, v, log_u, log_v, rep); });
}

int spk_sharded_info(const spk_sharded* S, int64_t* n, int64_t* nnz, int64_t* kernel_nnz, int64_t* lo, int64_t* hi,
                     int64_t* captured_launches) {
  if (!S) return SPK_STATUS_INPUT;
  if (n) *n = S->n;
  if (nnz) *nnz = S->nnz;
  if (kernel_nnz) *kernel_nnz = S->kernel_nnz;
  if (lo) *lo = S->lo;
  if (hi) *hi = S->hi;
  if (captured_launches) *captured_launches = S->graph ? S->g_launches : 0;
  return SPK_OK;
}

void spk_sharded_free(spk_sharded* S) {
  if (!S) return;
  spk_ctx* ctx = S->ctx;
  cudaSetDevice(ctx->device);
  AllocStreamScope scope(ctx->stream);
  delete S;
}

int spk_spar_sink_sharded(spk_comm* comm, const spk_kernel_desc* kd, const double* a, const double* b,
                          const spk_solver_cfg* cfg, double s, uint64_t seed, const spk_sketch_opts* opts, int uot,
                          double* u, double* v, double* log_u, double* log_v, spk_report* rep) {
  if (!comm || !comm->ctx || !cfg) return SPK_STATUS_INPUT;
  spk_sharded* S = nullptr;
  int rc = spk_sharded_build(comm, kd, a, b, plan_kind_of(opts, uot), cfg->lambda, cfg->epsilon, s, seed, opts, &S);
  if (rc == SPK_OK) rc = spk_sharded_solve(S, cfg, uot, u, v, log_u, log_v, rep);
  spk_sharded_free(S);
  return rc;
}

int spk_spar_sink_multi(const int* devices, int ndev, const spk_kernel_desc* kd, const double* a, const double* b,
                        const spk_solver_cfg* cfg, double s, uint64_t seed, const spk_sketch_opts* opts, int uot,
                        double* u, double* v, double* log_u, double* log_v, spk_report* rep) {
  if (!devices || ndev < 1 || !kd || !cfg) return SPK_STATUS_INPUT;
  std::vector<spk_ctx*> ctxs(ndev, nullptr);
  std::vector<spk_comm*> comms(ndev, nullptr);
  int rc = SPK_OK;
  for (int r = 0; r < ndev && rc == SPK_OK; ++r) rc = spk_ctx_create(devices[r], &ctxs[r]);
  if (rc == SPK_OK) rc = spk_comm_init_all(devices, ndev, ctxs.data(), comms.data());
  std::vector<int> rcs(ndev, SPK_OK);
  std::vector<std::string> msgs(ndev);
  if (rc == SPK_OK) {
    // one host thread per GPU; rank 0 writes the (identical) results
    std::vector<std::thread> th;
    for (int r = 0; r < ndev; ++r)
      th.emplace_back([&, r] {
        rcs[r] = spk_spar_sink_sharded(comms[r], kd, a, b, cfg, s, seed, opts, uot, r == 0 ? u : nullptr,
                                       r == 0 ? v : nullptr, r == 0 ? log_u : nullptr, r == 0 ? log_v : nullptr,
                                       r == 0 ? rep : nullptr);
      });
    for (auto& t : th) t.join();
    for (int r = 0; r < ndev && rc == SPK_OK; ++r) rc = rcs[r];
  }
  if (rc != SPK_OK) {  // keep the failing rank's error past its context (spk_last_error(NULL, ...))
    int cat = rc, kind = SPK_E_DEVICE;
    char buf[1024] = "spk_spar_sink_multi: device setup failed";
    for (int r = 0; r < ndev; ++r)
      if (ctxs[r] && (rcs[r] != SPK_OK || r == ndev - 1)) {
        if (rcs[r] != SPK_OK || ctxs[r]->err_category) spk_last_error(ctxs[r], &cat, &kind, buf, sizeof buf);
        if (rcs[r] != SPK_OK) break;
      }
    set_process_error(cat, kind, buf);
  }
  for (int r = 0; r < ndev; ++r) {
    spk_comm_destroy(comms[r]);
    spk_ctx_destroy(ctxs[r]);
  }
  return rc;
}

}  // extern "C"
