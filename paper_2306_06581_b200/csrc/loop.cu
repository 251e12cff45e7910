// loop.cu -- sparse half-step operator for the persistent Sinkhorn loop
// (north-star item 3).
//
// u-half: rows of the CSR sketch against v  (spmv,   proj/src/sparsify.cpp:203-213)
// v-half: columns of the CSC mirror against u (spmv_t, sparsify.cpp:215-226);
//         the CSC keeps rows ascending inside each column, i.e. the order
//         spmv_t accumulates them.
// log domain: kernel_log_apply(_t) (proj/src/solvers.cpp:96-136).
//
// Fast mode: one warp per row/column, coalesced index/value streams, the
// gathered scaling vector read through L2 (__ldcg: it is rewritten inside
// the same launch, so the non-coherent path is not allowed), FMA and a
// shuffle tree. Deterministic (parity) mode: one thread per output summing
// in index order with contraction-free dadd/dmul, bit-identical to the CPU.
#include <algorithm>
#include <cmath>
#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "loop_core.cuh"
#include "rowdot.cuh"

namespace spk {

namespace {

using loopcore::finalize_atom;

// One row's value by the G lanes of a group (fast mode): FMA sum of v * x,
// or the two-pass log-sum-exp; x read through L2 (rewritten in the launch).
// Every lane of the warp calls it (the group reductions are warp shuffles).
template <int G, bool LOG, class VT, bool XS = false>
__device__ __forceinline__ double group_row(const VT* __restrict__ val, const uint32_t* __restrict__ idx, int b, int e,
                                            const double* x, int gl) {
  if constexpr (!LOG) {
    // four independent index -> x chains in flight per lane (eight: no gain, 36.9k against 37.5k at C2)
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int p = b + gl;
    for (; p + 3 * G < e; p += 4 * G) {
      const uint32_t c0 = __ldg(idx + p), c1 = __ldg(idx + p + G), c2 = __ldg(idx + p + 2 * G),
                     c3 = __ldg(idx + p + 3 * G);
      const double w0 = (double)__ldg(val + p), w1 = (double)__ldg(val + p + G), w2 = (double)__ldg(val + p + 2 * G),
                   w3 = (double)__ldg(val + p + 3 * G);
      a0 = fma(w0, ld_x<XS>(x, c0), a0);
      a1 = fma(w1, ld_x<XS>(x, c1), a1);
      a2 = fma(w2, ld_x<XS>(x, c2), a2);
      a3 = fma(w3, ld_x<XS>(x, c3), a3);
    }
    for (; p < e; p += G) a0 = fma((double)__ldg(val + p), ld_x<XS>(x, __ldg(idx + p)), a0);
    double s = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int o = G / 2; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
  } else {
    double m = -CUDART_INF;
    for (int p = b + gl; p < e; p += G) {
      const double xv = ld_x<XS>(x, __ldg(idx + p));
      if (xv == -CUDART_INF) continue;
      m = fmax(m, log_of(ldg_val(val + p)) + xv);
    }
#pragma unroll
    for (int o = G / 2; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    double s = 0.0;
    if (m != -CUDART_INF)
      for (int p = b + gl; p < e; p += G) {
        const double xv = ld_x<XS>(x, __ldg(idx + p));
        if (xv == -CUDART_INF) continue;
        s += exp_term<VT>(log_of(ldg_val(val + p)) + xv - m);
      }
#pragma unroll
    for (int o = G / 2; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return m == -CUDART_INF ? -CUDART_INF : m + log(s);
  }
}

// G: lanes per row in fast mode (8 for short rows: 4 rows in flight per warp,
// the next rows' bounds loaded one step ahead; 32 for long rows).
// XS: the gathered vector staged in shared memory at the start of every half
// (n * 8 bytes per CTA; mid-size sketches, n <= kStageMaxN): each entry's x
// then costs a shared load instead of a second, dependent L2 round trip.
constexpr int64_t kStageMaxN = 24576;  // 192 KB of the one CTA per SM
template <class VT, int G = 32, bool XS = false>
struct SparseOp {
  // staged x: one 1024-thread CTA per SM (half the staging traffic and half
  // the grid-barrier participants of two 512-thread CTAs: C2 37.0k -> 40.5k)
  static constexpr int kThreads = XS ? 1024 : loopcore::kBlock;
  static constexpr int kMinBlocks = XS ? 1 : 2;
  int64_t n;
  const long long* row_ptr;
  const uint32_t* col_idx;
  const VT* val;
  const long long* col_ptr;
  const uint32_t* row_idx;
  const VT* val_t;

  template <int ROLE, bool LOG, bool DET>
  __device__ void half(const double* x, const double* wgt, const double* old, double* out, unsigned char* ne,
                       int* dyn, double exponent, int policy, int t, unsigned long long* flag, double* absdiff,
                       double& err, long long& masks) const {
    const long long* ptr = ROLE == 0 ? row_ptr : col_ptr;
    const uint32_t* idx = ROLE == 0 ? col_idx : row_idx;
    const VT* vv = ROLE == 0 ? val : val_t;
    const int lane = threadIdx.x & 31;
    if (XS && !DET) {
      extern __shared__ __align__(16) double x_stage[];
      __syncthreads();  // the previous half's readers are done
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x_stage[i] = __ldcg(x + i);
      __syncthreads();
      x = x_stage;
    }
    if (DET) {
      const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
      const int64_t nth = (int64_t)gridDim.x * blockDim.x;
      for (int64_t i = tid; i < n; i += nth) {
        double d = 0.0;
        const double o = __ldcg(old + i);
        if (ne[i]) {
          const double tmp = row_apply<LOG, true, VT>(vv, idx, ptr[i], ptr[i + 1], x, lane);
          d = finalize_atom<LOG>(i, tmp, o, wgt[i], exponent, policy, t, ne, dyn, out, flag, masks);
        } else {
          out[i] = o;
        }
        absdiff[i] = d;
      }
    } else if constexpr (G == 32) {
      const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
      const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
      for (int64_t i = warp; i < n; i += nw) {
        if (!ne[i]) {
          if (lane == 0) out[i] = __ldcg(old + i);
          continue;
        }
        const double tmp = row_apply<LOG, false, VT, XS>(vv, idx, __ldg(ptr + i), __ldg(ptr + i + 1), x, lane);
        if (lane == 0)
          err += finalize_atom<LOG>(i, tmp, __ldcg(old + i), __ldg(wgt + i), exponent, policy, t, ne, dyn, out, flag,
                                    masks);
      }
    } else {
      // 32 / G rows per warp at once (rows of ~50-200 entries: a warp per row
      // would leave its loads one L2 round trip at a time)
      constexpr int R = 32 / G;
      const int gl = lane & (G - 1);
      const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
      const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
      int64_t i = warp * R + lane / G;
      long long bn = 0, en = 0;
      if (i < n) {
        bn = __ldg(ptr + i);
        en = __ldg(ptr + i + 1);
      }
      for (int64_t i0 = warp * R; i0 < n; i0 += nw * R) {
        i = i0 + lane / G;
        const bool in = i < n;
        const bool live = in && ne[i];
        const long long b = live ? bn : 0, e = live ? en : 0;
        const int64_t inext = i + nw * R;
        if (inext < n) {  // the next rows' bounds in flight while this row runs
          bn = __ldg(ptr + inext);
          en = __ldg(ptr + inext + 1);
        }
        const VT* vr = vv + b;
        const uint32_t* ir = idx + b;
        const double tmp = group_row<G, LOG, VT, XS>(vr, ir, 0, (int)(e - b), x, gl);
        if (in && gl == 0) {
          if (!live) out[i] = __ldcg(old + i);
          else
            err += finalize_atom<LOG>(i, tmp, __ldcg(old + i), __ldg(wgt + i), exponent, policy, t, ne, dyn, out,
                                      flag, masks);
        }
      }
    }
  }
};

// kernel_coverage (solvers.cpp:154-163): rows from row_ptr, columns from col_ptr.
__global__ void coverage_kernel(const long long* row_ptr, const long long* col_ptr, int64_t n, unsigned char* row_ne,
                                unsigned char* col_ne, unsigned long long* empty) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned char r = row_ptr[i + 1] > row_ptr[i];
    const unsigned char c = col_ptr[i + 1] > col_ptr[i];
    row_ne[i] = r;
    col_ne[i] = c;
    if (!r) atomicAdd(&empty[0], 1ull);
    if (!c) atomicAdd(&empty[1], 1ull);
  }
}

template <bool LOG, class VT, int G, bool XS = false>
void run_g(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy, LoopState& st,
           LoopOut& out);

// fast mode on short rows (<= 256 entries on average): 8 lanes per row
template <bool LOG, class VT>
void run_t(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy, LoopState& st,
           LoopOut& out) {
  // auto: 8 lanes per row when rows are short AND a warp per row would leave
  // each warp several rows in sequence (measured: C5-sparse 13.5k -> 16.4k
  // iterations/s; C2, 10k rows = ~2 per warp, keeps a warp per row)
  const int64_t warps = (int64_t)ctx->num_sms * 2 * (loopcore::kBlock / 32);
  const bool stage = !ctx->deterministic && ctx->stage_x && sk->n <= kStageMaxN;
  // (with x staged in shared memory the 8-lane rows win at C2 too: 37.3k against 32.5k)
  const bool short_rows = ctx->row_lanes == 8 ||
                          (ctx->row_lanes == 0 && sk->nnz <= 256 * sk->n && (stage || sk->n > 4 * warps));
  if (!ctx->deterministic && short_rows) {
    if (stage) run_g<LOG, VT, 8, true>(ctx, sk, cfg, exponent, policy, st, out);
    else run_g<LOG, VT, 8>(ctx, sk, cfg, exponent, policy, st, out);
  } else if (stage) {
    run_g<LOG, VT, 32, true>(ctx, sk, cfg, exponent, policy, st, out);
  } else {
    run_g<LOG, VT, 32>(ctx, sk, cfg, exponent, policy, st, out);
  }
}

template <bool LOG, class VT, int G, bool XS>
void run_g(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy, LoopState& st,
           LoopOut& out) {
  const int64_t n = sk->n;
  LoopWs& W = sk->ws;
  W.row_ne.ensure(n);
  W.col_ne.ensure(n);
  SPK_CUDA(cudaMemcpyAsync(W.row_ne.p, sk->cov_row.p, n, cudaMemcpyDeviceToDevice, ctx->stream));
  SPK_CUDA(cudaMemcpyAsync(W.col_ne.p, sk->cov_col.p, n, cudaMemcpyDeviceToDevice, ctx->stream));
  SparseOp<VT, G, XS> op;
  op.n = n;
  op.row_ptr = sk->row_ptr.as<long long>();
  op.col_idx = sk->col_idx.as<uint32_t>();
  op.col_ptr = sk->col_ptr.as<long long>();
  op.row_idx = sk->row_idx.as<uint32_t>();
  if constexpr (std::is_same<VT, LogK>::value || std::is_same<VT, LogKf>::value) {  // log K~ precomputed once
    op.val = reinterpret_cast<const VT*>(sk->log_values.p);
    op.val_t = reinterpret_cast<const VT*>(sk->log_values_t.p);
  } else {
    op.val = sk->values.as<VT>();
    op.val_t = sk->values_t.as<VT>();
  }
  const int64_t per_block = ctx->deterministic ? loopcore::kBlock : loopcore::kBlock / G;
  // G = 8: every co-resident CTA (a grid just above the SM count would give
  // a few SMs two CTAs' rows and make every half wait for them)
  const int64_t useful = (!ctx->deterministic && G < 32) ? (int64_t)1 << 30 : (n + per_block - 1) / per_block;
  loopcore::run_core<LOG>(ctx, op, n, W, sk->cov_empty_rows, sk->cov_empty_cols, cfg, exponent, policy, st, useful,
                          out, /*exact_grid=*/0, XS ? sizeof(double) * (size_t)n : 0);
}

}  // namespace

namespace {

// spmv (sparsify.cpp:203-213) / spmv_t (:215-226, skipping x_i == 0) with
// one thread per output summing in index order.
template <class VT>
__global__ void product_kernel(int64_t n, const long long* ptr, const uint32_t* idx, const VT* val, const double* x,
                               double* y, int skip_zero) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (long long p = ptr[i]; p < ptr[i + 1]; ++p) {
      const double xv = x[idx[p]];
      if (skip_zero && xv == 0.0) continue;
      acc = dadd(acc, dmul((double)val[p], xv));
    }
    y[i] = acc;
  }
}

}  // namespace

void sketch_product(spk_ctx* ctx, spk_sketch* sk, const double* x_host, double* y_host, int transpose) {
  const int64_t n = sk->n;
  DBuf x, y(sizeof(double) * n);
  upload(ctx, x, x_host, sizeof(double) * n);
  const long long* ptr = transpose ? sk->col_ptr.as<long long>() : sk->row_ptr.as<long long>();
  const uint32_t* idx = transpose ? sk->row_idx.as<uint32_t>() : sk->col_idx.as<uint32_t>();
  const int g = loopcore::simple_grid(ctx, n);
  if (sk->value_type == SPK_VALUES_F32)
    product_kernel<float><<<g, 256, 0, ctx->stream>>>(n, ptr, idx, (transpose ? sk->values_t : sk->values).as<float>(),
                                                      x.as<double>(), y.as<double>(), transpose);
  else
    product_kernel<double><<<g, 256, 0, ctx->stream>>>(n, ptr, idx, (transpose ? sk->values_t : sk->values).as<double>(),
                                                       x.as<double>(), y.as<double>(), transpose);
  ++ctx->launches;
  download(ctx, y_host, y, sizeof(double) * n);
}

// kernel_coverage (solvers.cpp:154-163) of the sketch's structure: once per sketch.
void ensure_coverage(spk_ctx* ctx, spk_sketch* sk) {
  if (sk->cov_empty_rows >= 0) return;
  const int64_t n = sk->n;
  sk->cov_row.alloc(n);
  sk->cov_col.alloc(n);
  DBuf empty(16);
  SPK_CUDA(cudaMemsetAsync(empty.p, 0, 16, ctx->stream));
  coverage_kernel<<<loopcore::simple_grid(ctx, n), 256, 0, ctx->stream>>>(
      sk->row_ptr.as<long long>(), sk->col_ptr.as<long long>(), n, sk->cov_row.as<unsigned char>(),
      sk->cov_col.as<unsigned char>(), empty.as<unsigned long long>());
  ++ctx->launches;
  unsigned long long emp[2];
  download(ctx, emp, empty, sizeof emp);
  sk->cov_empty_rows = (long long)emp[0];
  sk->cov_empty_cols = (long long)emp[1];
}

template <class VT>
__global__ void log_values_kernel(const VT* v, int64_t m, double* out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
    out[k] = log((double)v[k]);
}

// log K~ of the CSR and CSC values (fp64 logs of the stored values: the same
// numbers the log-sum-exp took per entry before), built on the first
// log-domain solve of a sketch.
void ensure_log_values(spk_ctx* ctx, spk_sketch* sk) {
  if (sk->log_values.p) return;
  const int64_t m = std::max<int64_t>(sk->nnz, 1);
  sk->log_values.alloc(sizeof(double) * m);
  sk->log_values_t.alloc(sizeof(double) * m);
  if (sk->nnz == 0) return;
  const int g = loopcore::simple_grid(ctx, sk->nnz);
  if (sk->value_type == SPK_VALUES_F32) {
    log_values_kernel<float><<<g, 256, 0, ctx->stream>>>(sk->values.as<float>(), sk->nnz, sk->log_values.as<double>());
    log_values_kernel<float><<<g, 256, 0, ctx->stream>>>(sk->values_t.as<float>(), sk->nnz,
                                                         sk->log_values_t.as<double>());
  } else {
    log_values_kernel<double><<<g, 256, 0, ctx->stream>>>(sk->values.as<double>(), sk->nnz,
                                                          sk->log_values.as<double>());
    log_values_kernel<double><<<g, 256, 0, ctx->stream>>>(sk->values_t.as<double>(), sk->nnz,
                                                          sk->log_values_t.as<double>());
  }
  ctx->launches += 2;
}

void run_sparse_loop(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy,
                     LoopState& st, LoopOut& out) {
  const bool log_domain = cfg.stabilize != 0;
  NvtxRange nr(log_domain ? "spk:loop(log)" : "spk:loop");
  ensure_coverage(ctx, sk);
  // small sketches: one cluster, scalings in shared memory, no grid barriers
  if (run_cluster_loop(ctx, sk, cfg, exponent, policy, st, out)) return;
  // fast linear-domain path: slab x block layout with TMA-staged scalings
  // (auto: large sketches only; the layout pays off once x no longer sits in L1/L2-friendly sizes)
  // Mid-size sketches (n < 2^17): building the two layouts costs about as much
  // as the ~200 CSR iterations it would speed up (config 5: 5 ms against 23 us
  // saved per iteration), so a short first solve keeps the CSR loop and the
  // layout is built once the sketch is solved again or the budget is long.
  const bool mid = sk->n < (int64_t(1) << 17);
  const bool worth = !mid || sk->blocked_tried || sk->loop_solves > 0 || cfg.max_iter >= 400;
  ++sk->loop_solves;
  const bool try_blocked = ctx->use_blocked == 1 || (ctx->use_blocked == 2 && sk->n >= kBlockedAutoMinN && worth);
  if (!ctx->deterministic && !log_domain && try_blocked && run_blocked(ctx, sk, cfg, exponent, policy, st, out))
    return;
  if (log_domain) {
    ensure_log_values(ctx, sk);
    if (sk->value_type == SPK_VALUES_F32 && !ctx->deterministic) run_t<true, LogKf>(ctx, sk, cfg, exponent, policy, st, out);
    else run_t<true, LogK>(ctx, sk, cfg, exponent, policy, st, out);
  } else if (sk->value_type == SPK_VALUES_F32) {
    run_t<false, float>(ctx, sk, cfg, exponent, policy, st, out);
  } else {
    run_t<false, double>(ctx, sk, cfg, exponent, policy, st, out);
  }
}

}  // namespace spk
