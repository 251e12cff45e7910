// loop_core.cuh -- the Sinkhorn scaling loop as ONE persistent cooperative
// kernel, generic over the half-step operator (sparse sketch, dense K, or K
// recomputed on the fly from coordinates).
//
// Reference semantics: detail::scaling_loop (include/sparsink/solvers.hpp:256-395)
// and detail::log_scaling_loop (:397-513).
//
// One launch runs every iteration: u-half over rows, grid barrier, v-half
// over columns with the NEW u (Gauss-Seidel, :327), grid barrier, then every
// CTA reduces the per-CTA residual partials in the same fixed order and takes
// the same stop decision -- no host round trip per iteration. u and v are
// double-buffered, so "restore the previous iterate on divergence"
// (:321-325, :352-356) is just "do not flip the buffer".
#pragma once

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace spk {
namespace loopcore {

namespace cg = cooperative_groups;

constexpr unsigned long long kNone = ~0ull;
constexpr int kBlock = 512;

struct Part {
  double err;
  long long masks;
};

struct Status {
  long long iterations;
  int converged;
  int diverged;    // Mask policy blow-up (linear domain)
  int error_kind;  // SPK_E_* raised inside the loop (0 = none)
  int error_half;  // 0 = u-half (rows), 1 = v-half (cols)
  long long error_index;
  int cur;  // buffer index holding the final scalings
  int div_half;
  long long div_index;
  long long masked_rows_before, masked_cols_before, masks_u_last;
  long long masked_rows, masked_cols;
};

struct Common {
  int64_t n;
  const double* wa;  // a (linear) or log a (log domain)
  const double* wb;
  double* u0;
  double* u1;
  double* v0;
  double* v1;
  unsigned char* row_ne;
  unsigned char* col_ne;
  int* dyn_row;
  int* dyn_col;
  double* absdiff;           // 2n, deterministic-mode residual terms
  Part* part;                // [2 parity][2 halves][gridDim]
  unsigned long long* flag;  // [2 parity][2 halves] first bad index
  Status* status;
  long long max_iter;
  double delta;
  double exponent;
  int policy;
  long long masked_rows0, masked_cols0;
};

// The per-atom update of one half (solvers.hpp:292-320 / :438-450).
// Returns the residual term |new - old| (0 when the atom leaves the sum).
template <bool LOG>
__device__ __forceinline__ double finalize_atom(int64_t i, double tmp, double old, double w, double exponent,
                                                int policy, int t, unsigned char* ne, int* dyn, double* out,
                                                unsigned long long* flag, long long& masks) {
  if (!LOG) {
    if (tmp <= 0.0 || !isfinite(tmp)) {
      if (policy == SPK_POLICY_MASK && tmp == 0.0) {  // dynamic mask (:296-301)
        ne[i] = 0;
        dyn[i] = t;
        out[i] = 0.0;
        ++masks;
        return fabs(0.0 - old);
      }
      atomicMin(flag, (unsigned long long)i);  // diverged (Mask) / ZeroDenominator (Error)
      out[i] = old;
      return 0.0;
    }
    const double q = w / tmp;
    const double un = (exponent == 1.0) ? q : pow(q, exponent);
    if (!(un <= 1e150) && policy == SPK_POLICY_MASK) atomicMin(flag, (unsigned long long)i);  // :316-319
    out[i] = un;
    return fabs(un - old);
  } else {
    if (tmp == -CUDART_INF) {
      if (policy == SPK_POLICY_MASK) {  // :440-446
        ne[i] = 0;
        dyn[i] = t;
        out[i] = -CUDART_INF;
        ++masks;
        return 0.0;  // masked atoms leave the log residual (:472-475)
      }
      atomicMin(flag, (unsigned long long)i);
      out[i] = old;
      return 0.0;
    }
    const double ln = exponent * (w - tmp);  // :449
    out[i] = ln;
    return fabs(ln - old);
  }
}

// Block reduction of (err, masks) into slot[blockIdx.x].
__device__ inline void block_partial(double err, long long masks, Part* slot) {
  __shared__ double se[32];
  __shared__ long long sm[32];
  err = warp_sum(err);
  masks = warp_sum_ll(masks);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    se[w] = err;
    sm[w] = masks;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double e = 0.0;
    long long m = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      e += se[k];
      m += sm[k];
    }
    slot[blockIdx.x].err = e;
    slot[blockIdx.x].masks = m;
  }
  __syncthreads();
}

// Fixed-order reduction of the per-CTA partials; every CTA gets the same value.
__device__ inline void reduce_parts(const Part* p, int nb, double& err, long long& masks) {
  __shared__ double re;
  __shared__ long long rm;
  if (threadIdx.x < 32) {
    double e = 0.0;
    long long m = 0;
    for (int k = threadIdx.x; k < nb; k += 32) {
      e += __ldcg(&p[k].err);
      m += __ldcg(&p[k].masks);
    }
    e = warp_sum(e);
    m = warp_sum_ll(m);
    if (threadIdx.x == 0) {
      re = e;
      rm = m;
    }
  }
  __syncthreads();
  err = re;
  masks = rm;
  __syncthreads();
}

// Op must provide:
//   template <int ROLE, bool LOG, bool DET> __device__ void half(
//       const double* x, const double* wgt, const double* old, double* out,
//       unsigned char* ne, int* dyn, double exponent, int policy, int t,
//       unsigned long long* flag, double* absdiff, double& err, long long& masks) const;
// ROLE 0 = rows of K (u-half, x = v), ROLE 1 = columns (v-half, x = u).
template <bool LOG, bool DET, class Op>
__global__ void __launch_bounds__(Op::kThreads, Op::kMinBlocks) loop_kernel(Common P, Op op) {
  cg::grid_group grid = cg::this_grid();
  const int nb = gridDim.x;
  double* U[2] = {P.u0, P.u1};
  double* V[2] = {P.v0, P.v1};
  int cur = 0;
  long long mr = P.masked_rows0, mc = P.masked_cols0;
  long long t = 0;
  int converged = 0, diverged = 0, ekind = 0, ehalf = 0, dhalf = 0;
  long long eidx = 0, didx = 0, mr_before = mr, mc_before = mc, mu_last = 0;
  while (t < P.max_iter) {
    ++t;
    const int par = (int)(t & 1);
    const int nxt = cur ^ 1;
    Part* part_u = P.part + (size_t)(par * 2 + 0) * nb;
    Part* part_v = P.part + (size_t)(par * 2 + 1) * nb;
    unsigned long long* flag_u = P.flag + par * 2 + 0;
    unsigned long long* flag_v = P.flag + par * 2 + 1;
    mr_before = mr;
    mc_before = mc;

    // ---- u-half: u_i from (K v)_i ----
    double err = 0.0;
    long long masks = 0;
    op.template half<0, LOG, DET>(V[cur], P.wa, U[cur], U[nxt], P.row_ne, P.dyn_row, P.exponent, P.policy, (int)t,
                                  flag_u, P.absdiff, err, masks);
    block_partial(err, masks, part_u);
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // recycle the other parity's flags for t+1
      P.flag[(par ^ 1) * 2 + 0] = kNone;
      P.flag[(par ^ 1) * 2 + 1] = kNone;
    }
    const unsigned long long fu = __ldcg(flag_u);
    double err_u;
    long long masks_u;
    reduce_parts(part_u, nb, err_u, masks_u);
    if (fu != kNone) {
      if (P.policy == SPK_POLICY_MASK && !LOG) {
        diverged = 1;
        dhalf = 0;
        didx = (long long)fu;
      } else {
        ekind = SPK_E_ZERO_DENOMINATOR;
        ehalf = 0;
        eidx = (long long)fu;
      }
      mu_last = 0;
      break;
    }

    // ---- v-half: v_j from (K' u_new)_j ----
    err = 0.0;
    masks = 0;
    op.template half<1, LOG, DET>(U[nxt], P.wb, V[cur], V[nxt], P.col_ne, P.dyn_col, P.exponent, P.policy, (int)t,
                                  flag_v, P.absdiff + P.n, err, masks);
    block_partial(err, masks, part_v);
    grid.sync();
    const unsigned long long fv = __ldcg(flag_v);
    double err_v;
    long long masks_v;
    reduce_parts(part_v, nb, err_v, masks_v);
    if (fv != kNone) {
      if (P.policy == SPK_POLICY_MASK && !LOG) {
        diverged = 1;
        dhalf = 1;
        didx = (long long)fv;
      } else {
        ekind = SPK_E_ZERO_DENOMINATOR;
        ehalf = 1;
        eidx = (long long)fv;
      }
      mu_last = masks_u;
      break;
    }
    mr += masks_u;
    mc += masks_v;
    cur = nxt;
    if (mr == P.n || mc == P.n) {  // solvers.hpp:357-358 / :465-466
      ekind = SPK_E_DEGENERATE_SKETCH_ERROR;
      break;
    }
    if (t >= 2) {
      double e;
      if (DET) {  // sequential sum in index order (:361-363 / :471-475)
        __shared__ double se;
        if (threadIdx.x == 0) {
          double acc = 0.0;
          for (int64_t k = 0; k < 2 * P.n; ++k) acc = dadd(acc, __ldcg(P.absdiff + k));
          se = acc;
        }
        __syncthreads();
        e = se;
        __syncthreads();
      } else {
        e = err_u + err_v;
      }
      if (e <= P.delta) {
        converged = 1;
        break;
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Status* s = P.status;
    s->iterations = t;
    s->converged = converged;
    s->diverged = diverged;
    s->error_kind = ekind;
    s->error_half = ehalf;
    s->error_index = eidx;
    s->cur = cur;
    s->div_half = dhalf;
    s->div_index = didx;
    s->masked_rows_before = mr_before;
    s->masked_cols_before = mc_before;
    s->masks_u_last = mu_last;
    s->masked_rows = mr;
    s->masked_cols = mc;
  }
}

// ---- setup / epilogue kernels ---------------------------------------------------

template <bool LOG>
__global__ void init_scalings_kernel(int64_t n, const unsigned char* row_ne, const unsigned char* col_ne, double* u,
                                     double* v) {
  // u = v = 1 on covered atoms, 0 (log: 0 / -inf) elsewhere (:277-281, :424-428)
  const double on = LOG ? 0.0 : 1.0;
  const double off = LOG ? -CUDART_INF : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    u[i] = row_ne[i] ? on : off;
    v[i] = col_ne[i] ? on : off;
  }
}

static __global__ void log_weights_kernel(int64_t n, const double* a, double* la) {  // :417-421
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    la[i] = a[i] > 0.0 ? log(a[i]) : -CUDART_INF;
}

static __global__ void count_dyn_kernel(const int* dyn, int64_t n, int t, long long limit, unsigned long long* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (dyn[i] == t && i < limit) atomicAdd(out, 1ull);
}

static __global__ void exp_kernel(int64_t n, const double* l, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = exp(l[i]);
}

static __global__ void fill_u64_kernel(unsigned long long* p, int m, unsigned long long v) {
  if ((int)threadIdx.x < m) p[threadIdx.x] = v;
}

static __global__ void zero_int_kernel(int* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0;
}

inline int simple_grid(spk_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8));
}

// Opt a kernel into the largest dynamic shared memory the device allows
// (not the launch's own size: contexts on other host threads launch the same
// kernel with other sizes, and a smaller attribute set between another
// thread's set and launch would fail that launch).
inline void allow_max_dyn_smem(const void* kern) {
  int dev = 0, optin = 0;
  SPK_CUDA(cudaGetDevice(&dev));
  SPK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa{};
  SPK_CUDA(cudaFuncGetAttributes(&fa, kern));
  SPK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes));
}

// Cluster size an operator asks for (Op::kCluster, default 1).
template <class Op, class = void>
struct cluster_of {
  static constexpr int value = 1;
};
template <class Op>
struct cluster_of<Op, std::void_t<decltype(Op::kCluster)>> {
  static constexpr int value = Op::kCluster;
};

template <bool LOG>
void loop_epilogue(spk_ctx* ctx, const Status& S, int64_t n, LoopWs& W, const double* uf, const double* vf,
                   LoopState& st, LoopOut& out);

// Host driver shared by every operator. row_ne / col_ne hold the structural
// coverage (kernel_coverage, solvers.cpp:138-163); masked_rows/cols their
// zero counts. Fills st.u/st.v (and st.lu/st.lv in the log domain).
// exact_grid > 0 demands exactly that many co-resident CTAs (one slab each);
// dyn_smem is the operator's dynamic shared memory per CTA.
template <bool LOG, class Op>
void run_core(spk_ctx* ctx, const Op& op, int64_t n, LoopWs& W, long long masked_rows, long long masked_cols,
              const spk_solver_cfg& cfg, double exponent, int policy, LoopState& st, int64_t useful_blocks,
              LoopOut& out, int exact_grid = 0, size_t dyn_smem = 0) {
  cudaStream_t s = ctx->stream;
  const int64_t npad = (n + 15) & ~int64_t(15);  // 128-byte aligned ping-pong halves (TMA sources)
  DBuf& row_ne = W.row_ne;
  DBuf& col_ne = W.col_ne;
  // solvers.hpp:269-274 / :411-414
  if ((masked_rows || masked_cols) && policy == SPK_POLICY_ERROR) {
    if (LOG) fail(SPK_E_ZERO_DENOMINATOR, "kernel has empty rows or columns");
    fail(SPK_E_ZERO_DENOMINATOR, "kernel has " + std::to_string(masked_rows) + " empty rows and " +
                                     std::to_string(masked_cols) + " empty columns");
  }
  if (masked_rows == n || masked_cols == n) fail(SPK_E_DEGENERATE_SKETCH_ERROR, "kernel has no entries at all");

  W.dyn_row.ensure(sizeof(int) * n);
  W.dyn_col.ensure(sizeof(int) * n);
  W.u2.ensure(sizeof(double) * (2 * npad + 16));
  W.v2.ensure(sizeof(double) * (2 * npad + 16));
  W.absdiff.ensure(sizeof(double) * 2 * n);
  DBuf& dyn_row = W.dyn_row;
  DBuf& dyn_col = W.dyn_col;
  DBuf& u2 = W.u2;
  DBuf& v2 = W.v2;
  DBuf& absdiff = W.absdiff;
  SPK_CUDA(cudaMemsetAsync(dyn_row.p, 0, sizeof(int) * n, s));
  SPK_CUDA(cudaMemsetAsync(dyn_col.p, 0, sizeof(int) * n, s));
  const double* wa = st.a;
  const double* wb = st.b;
  if (LOG) {
    W.la.ensure(sizeof(double) * n);
    W.lb.ensure(sizeof(double) * n);
    log_weights_kernel<<<simple_grid(ctx, n), 256, 0, s>>>(n, st.a, W.la.as<double>());
    log_weights_kernel<<<simple_grid(ctx, n), 256, 0, s>>>(n, st.b, W.lb.as<double>());
    ctx->launches += 2;
    wa = W.la.as<double>();
    wb = W.lb.as<double>();
  }
  init_scalings_kernel<LOG><<<simple_grid(ctx, n), 256, 0, s>>>(n, row_ne.as<unsigned char>(),
                                                               col_ne.as<unsigned char>(), u2.as<double>(),
                                                               v2.as<double>());
  ++ctx->launches;

  // grid: co-resident CTAs (cooperative), no more than useful
  const bool det = ctx->deterministic != 0;
  auto kern = det ? loop_kernel<LOG, true, Op> : loop_kernel<LOG, false, Op>;
  if (dyn_smem > 0)
    allow_max_dyn_smem((const void*)kern);
  int per_sm = 0;
  SPK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Op::kThreads, dyn_smem));
  if (per_sm < 1) fail_device("loop_kernel occupancy", cudaErrorLaunchOutOfResources);
  if (ctx->loop_blocks_per_sm > 0) per_sm = std::min(per_sm, ctx->loop_blocks_per_sm);
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->num_sms * per_sm, useful_blocks));
  if (exact_grid > 0) {
    if ((int64_t)ctx->num_sms * per_sm < exact_grid)
      fail_device("loop_kernel: slabs exceed co-resident CTAs", cudaErrorCooperativeLaunchTooLarge);
    grid = exact_grid;
  }

  W.part.ensure(sizeof(Part) * 4 * grid);
  W.flag.ensure(sizeof(unsigned long long) * 4);
  W.status.ensure(sizeof(Status));
  DBuf& part = W.part;
  DBuf& flag = W.flag;
  DBuf& status = W.status;
  fill_u64_kernel<<<1, 32, 0, s>>>(flag.as<unsigned long long>(), 4, kNone);
  ++ctx->launches;
  SPK_CUDA(cudaMemsetAsync(status.p, 0, sizeof(Status), s));

  Common P{};
  P.n = n;
  P.wa = wa;
  P.wb = wb;
  P.u0 = u2.as<double>();
  P.u1 = u2.as<double>() + npad;
  P.v0 = v2.as<double>();
  P.v1 = v2.as<double>() + npad;
  P.row_ne = row_ne.as<unsigned char>();
  P.col_ne = col_ne.as<unsigned char>();
  P.dyn_row = dyn_row.as<int>();
  P.dyn_col = dyn_col.as<int>();
  P.absdiff = absdiff.as<double>();
  P.part = part.as<Part>();
  P.flag = flag.as<unsigned long long>();
  P.status = status.as<Status>();
  P.max_iter = cfg.max_iter;
  P.delta = cfg.delta;
  P.exponent = exponent;
  P.policy = policy;
  P.masked_rows0 = masked_rows;
  P.masked_cols0 = masked_cols;

  Op op_copy = op;
  void* args[] = {&P, &op_copy};
  Timer tm(s);
  if (cluster_of<Op>::value > 1) {  // cooperative launch of 2-CTA clusters (grid.sync + DSMEM)
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(Op::kThreads);
    lc.dynamicSmemBytes = dyn_smem;
    lc.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cluster_of<Op>::value;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 2;
    SPK_CUDA(cudaLaunchKernelExC(&lc, (const void*)kern, args));
  } else {
    SPK_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(Op::kThreads), args, dyn_smem, s));
  }
  ++ctx->launches;
  out.loop_s = tm.stop();
  SPK_CUDA(cudaGetLastError());
  Status S;
  download(ctx, &S, status, sizeof S);
  loop_epilogue<LOG>(ctx, S, n, W, u2.as<double>() + (size_t)S.cur * npad, v2.as<double>() + (size_t)S.cur * npad, st,
                     out);
}

// Loop outcome -> LoopOut (raising the loop's failures) and the final
// scalings uf / vf (device, n each) -> st.u / st.v (+ st.lu / st.lv).
template <bool LOG>
void loop_epilogue(spk_ctx* ctx, const Status& S, int64_t n, LoopWs& W, const double* uf, const double* vf,
                   LoopState& st, LoopOut& out) {
  cudaStream_t s = ctx->stream;
  DBuf& dyn_row = W.dyn_row;
  DBuf& dyn_col = W.dyn_col;
  if (S.error_kind == SPK_E_ZERO_DENOMINATOR) {
    const std::string idx = std::to_string(S.error_index);
    if (LOG)
      fail(SPK_E_ZERO_DENOMINATOR, S.error_half == 0 ? "Kv vanished at row " + idx : "K'u vanished at column " + idx);
    fail(SPK_E_ZERO_DENOMINATOR, S.error_half == 0
                                     ? "Kv underflowed at row " + idx + "; consider SolverConfig::stabilize"
                                     : "K'u underflowed at column " + idx + "; consider SolverConfig::stabilize");
  }
  if (S.error_kind == SPK_E_DEGENERATE_SKETCH_ERROR) fail(SPK_E_DEGENERATE_SKETCH_ERROR, "masking removed every atom");

  out.iterations = S.iterations;
  out.converged = S.converged;
  out.diverged = S.diverged;
  if (S.diverged) {
    // Only dynamic masks met before the first diverging index count: the
    // reference breaks out of its sequential sweep there (:306-307).
    DBuf cnt(sizeof(unsigned long long));
    SPK_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes, s));
    count_dyn_kernel<<<simple_grid(ctx, n), 256, 0, s>>>(S.div_half == 0 ? dyn_row.as<int>() : dyn_col.as<int>(), n,
                                                        (int)S.iterations, S.div_index, cnt.as<unsigned long long>());
    ++ctx->launches;
    unsigned long long c = 0;
    download(ctx, &c, cnt, sizeof c);
    if (S.div_half == 0) {
      out.masked_rows = S.masked_rows_before + (long long)c;
      out.masked_cols = S.masked_cols_before;
    } else {
      out.masked_rows = S.masked_rows_before + S.masks_u_last;
      out.masked_cols = S.masked_cols_before + (long long)c;
    }
  } else {
    out.masked_rows = S.masked_rows;
    out.masked_cols = S.masked_cols;
  }
  st.u->ensure(sizeof(double) * n);
  st.v->ensure(sizeof(double) * n);
  if (LOG) {
    st.lu->ensure(sizeof(double) * n);
    st.lv->ensure(sizeof(double) * n);
    SPK_CUDA(cudaMemcpyAsync(st.lu->p, uf, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    SPK_CUDA(cudaMemcpyAsync(st.lv->p, vf, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    exp_kernel<<<simple_grid(ctx, n), 256, 0, s>>>(n, st.lu->as<double>(), st.u->as<double>());
    exp_kernel<<<simple_grid(ctx, n), 256, 0, s>>>(n, st.lv->as<double>(), st.v->as<double>());
    ctx->launches += 2;
  } else {
    SPK_CUDA(cudaMemcpyAsync(st.u->p, uf, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    SPK_CUDA(cudaMemcpyAsync(st.v->p, vf, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }
  SPK_CUDA(cudaStreamSynchronize(s));
}

}  // namespace loopcore
}  // namespace spk
