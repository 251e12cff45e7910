// batch.cu -- many small log-domain Sparse Sinkhorn solves at once (config 3:
// 496 WFR frame pairs of n = 12,544, each run by pairwise_wfr,
// proj/src/harness.cpp:349-406, one spar_sink_uot at a time).
//
// One CTA owns one sketch for its whole solve: both log scalings (lu, lv:
// 2 n fp64 = 196 KB at n = 12,544) live in shared memory for every
// iteration, so the gathered x of a half is a shared-memory read and the
// only HBM traffic is the sketch stream (indices + log K~). CTAs are
// independent (no grid barrier): the grid is the batch, run in waves.
//
// Semantics: detail::log_scaling_loop (include/sparsink/solvers.hpp:397-513),
// as the single-sketch fast path (two-pass log-sum-exp; the sums run in
// another lane order, so scalings agree to rounding): lu = f (log a - LSE_j(log K~ +
// lv)); a row whose LSE is -inf is masked (Mask) or raises ZeroDenominator
// (Error); the stop rule sums |d lu| + |d lv| over unmasked atoms for t >= 2;
// all rows or all columns masked raises DegenerateSketchError.
#include <algorithm>
#include <cmath>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "loop_core.cuh"
#include "rowdot.cuh"

namespace spk {

namespace {

constexpr int kBatchThreads = 1024;

struct BatchItem {
  int64_t n;
  const long long* row_ptr;
  const uint32_t* col_idx;
  const double* lval;  // log K~ of the CSR values
  const long long* col_ptr;
  const uint32_t* row_idx;
  const double* lval_t;  // log K~ of the CSC values
  const double* la;      // log a (-inf where a = 0)
  const double* lb;
  const unsigned char* cov_row;  // structural coverage (kernel_coverage)
  const unsigned char* cov_col;
  double* lu;  // final log scalings (device, n each)
  double* lv;
  long long masked_rows0, masked_cols0;
  double exponent;
};

struct BatchStatus {
  long long iterations;
  long long masked_rows, masked_cols;
  long long error_index;
  int converged, error_kind, error_half, pad;
};

struct BatchArgs {
  const BatchItem* items;
  BatchStatus* status;
  long long max_iter;
  double delta;
  int policy;
  int npad;  // shared doubles per vector
};

// One half: out[i] for every unmasked output atom i from the row/column
// [ptr[i], ptr[i+1]) against the shared vector x. Returns this thread's
// residual share; masks and the first failing atom go through shared counters.
// Rows are short (config 3: ~94 entries), so 8 lanes share a row (4 rows per
// warp) and each lane keeps 4 independent entry loads in flight: the pass is
// bound by the latency of the sketch stream, not by its exp()s.
// Two-pass log-sum-exp (max, then the sum of exp(t - max): the reference's
// order, solvers.cpp:99-111).
constexpr int kG = 8;  // lanes per row

__device__ __forceinline__ double group_max(double v) {
#pragma unroll
  for (int o = kG / 2; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = kG / 2; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <class VT>
__device__ __forceinline__ double batch_half(int64_t n, const long long* __restrict__ ptr,
                                             const uint32_t* __restrict__ idx, const double* __restrict__ lval,
                                             const double* __restrict__ w, const double* x, double* out,
                                             unsigned int* ne, double exponent, int policy, long long* masks,
                                             unsigned long long* bad) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & (kG - 1);
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  constexpr int kRows = 32 / kG;
  constexpr bool kOnline = std::is_same<VT, LogKf>::value;
  double err = 0.0;
  // row bounds of the next row group loaded one group ahead
  int64_t i = (int64_t)warp * kRows + (lane / kG);
  long long bn = 0, en = 0;
  if (i < n) {
    bn = __ldg(ptr + i);
    en = __ldg(ptr + i + 1);
  }
  for (int64_t i0 = (int64_t)warp * kRows; i0 < n; i0 += (int64_t)nw * kRows) {
    i = i0 + (lane / kG);
    const bool live = i < n && ((ne[i >> 5] >> (i & 31)) & 1u);  // masked rows keep -inf
    long long b = live ? bn : 0, e = live ? en : 0;
    {
      const int64_t inext = i + (int64_t)nw * kRows;
      if (inext < n) {
        bn = __ldg(ptr + inext);
        en = __ldg(ptr + inext + 1);
      }
    }
    double m = -CUDART_INF, s = 0.0;
    if (kOnline) {
      // fp32 sketches: one pass, online (max, scaled sum) with the fp32-accurate
      // exp (each term rescaled at most once per new max)
      long long p = b + gl;
      auto add = [&](double t) {
        if (t == -CUDART_INF) return;
        if (t > m) {
          s = s * exp_fast(m - t) + 1.0;
          m = t;
        } else {
          s += exp_fast(t - m);
        }
      };
      for (; p + 3 * kG < e; p += 4 * kG) {
        uint32_t j[4];
        double l[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          j[k] = __ldg(idx + p + k * kG);
          l[k] = __ldg(lval + p + k * kG);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double xv = x[j[k]];
          if (xv != -CUDART_INF) add(l[k] + xv);
        }
      }
      for (; p < e; p += kG) {
        const double xv = x[__ldg(idx + p)];
        if (xv != -CUDART_INF) add(__ldg(lval + p) + xv);
      }
#pragma unroll
      for (int o = kG / 2; o; o >>= 1) {
        const double m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const double s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const double M = fmax(m, m2);
        if (M != -CUDART_INF)
          s = (m == -CUDART_INF ? 0.0 : s * exp_fast(m - M)) + (m2 == -CUDART_INF ? 0.0 : s2 * exp_fast(m2 - M));
        m = M;
      }
    } else {
      // fp64 sketches: two passes (max, then the sum of exp(t - max): the
      // reference's order, solvers.cpp:99-111)
      long long p = b + gl;
      for (; p + 3 * kG < e; p += 4 * kG) {
        uint32_t j[4];
        double l[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          j[k] = __ldg(idx + p + k * kG);
          l[k] = __ldg(lval + p + k * kG);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double xv = x[j[k]];
          if (xv != -CUDART_INF) m = fmax(m, l[k] + xv);
        }
      }
      for (; p < e; p += kG) {
        const double xv = x[__ldg(idx + p)];
        if (xv != -CUDART_INF) m = fmax(m, __ldg(lval + p) + xv);
      }
      m = group_max(m);
      if (m != -CUDART_INF) {
        p = b + gl;
        for (; p + 3 * kG < e; p += 4 * kG) {
          uint32_t j[4];
          double l[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            j[k] = __ldg(idx + p + k * kG);
            l[k] = __ldg(lval + p + k * kG);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double xv = x[j[k]];
            if (xv != -CUDART_INF) s += exp(l[k] + xv - m);
          }
        }
        for (; p < e; p += kG) {
          const double xv = x[__ldg(idx + p)];
          if (xv != -CUDART_INF) s += exp(__ldg(lval + p) + xv - m);
        }
      }
      s = group_sum(s);
    }
    {  // the next row's entry ranges into L2 while this row finishes (its bounds have arrived by now)
      const int64_t inext = i + (int64_t)nw * kRows;
      if (inext < n && en > bn) {
        const char* i0p = reinterpret_cast<const char*>(idx + bn);
        const char* l0p = reinterpret_cast<const char*>(lval + bn);
        const long long li = ((long long)(en - bn) * 4 + 127) >> 7, ll = ((long long)(en - bn) * 8 + 127) >> 7;
        for (long long q = gl; q < li + ll; q += kG) {
          const char* a = q < li ? i0p + (q << 7) : l0p + ((q - li) << 7);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
        }
      }
    }
    if (live && gl == 0) {
      const double lse = m == -CUDART_INF ? -CUDART_INF : m + log(s);
      if (lse == -CUDART_INF) {
        if (policy == SPK_POLICY_MASK) {  // :440-446 (masked atoms leave the residual)
          atomicAnd(ne + (i >> 5), ~(1u << (i & 31)));
          out[i] = -CUDART_INF;
          atomicAdd(reinterpret_cast<unsigned long long*>(masks), 1ull);
        } else {
          atomicMin(bad, (unsigned long long)i);
        }
      } else {
        const double ln = exponent * (__ldg(w + i) - lse);  // :449
        err += fabs(ln - out[i]);
        out[i] = ln;
      }
    }
  }
  return err;
}

// Fixed-order CTA sum (warp sums, then warp 0 over the warps in order).
__device__ __forceinline__ double cta_sum(double v, double* scratch) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double r = 0.0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) r += scratch[k];
  return r;
}

// VT: LogK (fp64 exp) or LogKf (fp32 sketches: fp32-accurate exp), as the single-sketch path
template <class VT>
__global__ void __launch_bounds__(kBatchThreads, 1) batch_log_kernel(BatchArgs A) {
  extern __shared__ __align__(16) double smem[];
  const BatchItem& I = A.items[blockIdx.x];
  const int64_t n = I.n;
  double* lu = smem;
  double* lv = smem + A.npad;
  unsigned int* neu = reinterpret_cast<unsigned int*>(lv + A.npad);
  unsigned int* nev = neu + (A.npad >> 5);
  __shared__ double scratch[32];
  __shared__ long long masks_sh[2];
  __shared__ unsigned long long bad_sh[2];
  // u = v = 1 (log 0) on covered atoms, masked atoms -inf (:424-428)
  for (int64_t w = threadIdx.x; w < (A.npad >> 5); w += blockDim.x) {
    unsigned int bu = 0u, bv = 0u;
    for (int k = 0; k < 32; ++k) {
      const int64_t i = w * 32 + k;
      if (i < n) {
        bu |= (I.cov_row[i] ? 1u : 0u) << k;
        bv |= (I.cov_col[i] ? 1u : 0u) << k;
      }
    }
    neu[w] = bu;
    nev[w] = bv;
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    lu[i] = I.cov_row[i] ? 0.0 : -CUDART_INF;
    lv[i] = I.cov_col[i] ? 0.0 : -CUDART_INF;
  }
  long long mr = I.masked_rows0, mc = I.masked_cols0;
  long long t = 0;
  int converged = 0, ekind = 0, ehalf = 0;
  long long eidx = 0;
  __syncthreads();
  while (t < A.max_iter) {
    ++t;
    __syncthreads();  // every thread has read last iteration's counters
    if (threadIdx.x == 0) {
      masks_sh[0] = masks_sh[1] = 0;
      bad_sh[0] = bad_sh[1] = ~0ull;
    }
    __syncthreads();
    // u-half: rows of K~ against lv (kernel_log_apply, solvers.cpp:96-116)
    const double eu = cta_sum(
        batch_half<VT>(n, I.row_ptr, I.col_idx, I.lval, I.la, lv, lu, neu, I.exponent, A.policy, &masks_sh[0], &bad_sh[0]),
        scratch);
    __syncthreads();
    if (bad_sh[0] != ~0ull) {
      ekind = SPK_E_ZERO_DENOMINATOR;
      ehalf = 0;
      eidx = (long long)bad_sh[0];
      break;
    }
    // v-half: columns against the NEW lu (Gauss-Seidel, :451-463)
    const double ev = cta_sum(
        batch_half<VT>(n, I.col_ptr, I.row_idx, I.lval_t, I.lb, lu, lv, nev, I.exponent, A.policy, &masks_sh[1],
                   &bad_sh[1]),
        scratch);
    __syncthreads();
    if (bad_sh[1] != ~0ull) {
      ekind = SPK_E_ZERO_DENOMINATOR;
      ehalf = 1;
      eidx = (long long)bad_sh[1];
      break;
    }
    mr += masks_sh[0];
    mc += masks_sh[1];
    if (mr == n || mc == n) {  // :465-466
      ekind = SPK_E_DEGENERATE_SKETCH_ERROR;
      break;
    }
    if (t >= 2 && eu + ev <= A.delta) {  // :468-480
      converged = 1;
      break;
    }
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    I.lu[i] = lu[i];
    I.lv[i] = lv[i];
  }
  if (threadIdx.x == 0) {
    BatchStatus& S = A.status[blockIdx.x];
    S.iterations = t;
    S.masked_rows = mr;
    S.masked_cols = mc;
    S.converged = converged;
    S.error_kind = ekind;
    S.error_half = ehalf;
    S.error_index = eidx;
  }
}

__global__ void exp_pair_kernel(int64_t n, const double* lu, const double* lv, double* u, double* v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    u[i] = exp(lu[i]);
    v[i] = exp(lv[i]);
  }
}

}  // namespace

// Largest sketch dimension one CTA can hold (both log scalings + mask bits).
int64_t batch_max_n(spk_ctx* ctx) {
  int optin = 0;
  SPK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const int64_t avail = (int64_t)optin - 1024;  // static shared use
  // per atom: 2 doubles + 2 bits
  return std::max<int64_t>(0, (avail * 8 / (2 * 64 + 2)) / 32 * 32 - 32);
}

// The batched loop over sks[0..count); returns per-item loop outcomes.
void run_batch_log(spk_ctx* ctx, spk_sketch* const* sks, int count, const spk_solver_cfg& cfg,
                   const std::vector<double>& exponents, int policy, std::vector<LoopOut>& outs,
                   std::vector<std::string>& errors, std::vector<int>& error_kinds) {
  cudaStream_t s = ctx->stream;
  int64_t nmax = 0;
  for (int k = 0; k < count; ++k) nmax = std::max(nmax, sks[k]->n);
  const int npad = (int)((nmax + 31) / 32 * 32);
  std::vector<BatchItem> items(count);
  for (int k = 0; k < count; ++k) {
    spk_sketch* sk = sks[k];
    const int64_t n = sk->n;
    ensure_coverage(ctx, sk);
    ensure_log_values(ctx, sk);
    LoopWs& W = sk->ws;
    W.la.ensure(sizeof(double) * n);
    W.lb.ensure(sizeof(double) * n);
    loopcore::log_weights_kernel<<<loopcore::simple_grid(ctx, n), 256, 0, s>>>(n, sk->a.as<double>(),
                                                                              W.la.as<double>());
    loopcore::log_weights_kernel<<<loopcore::simple_grid(ctx, n), 256, 0, s>>>(n, sk->b.as<double>(),
                                                                              W.lb.as<double>());
    ctx->launches += 2;
    sk->lu.ensure(sizeof(double) * n);
    sk->lv.ensure(sizeof(double) * n);
    BatchItem& I = items[k];
    I.n = n;
    I.row_ptr = sk->row_ptr.as<long long>();
    I.col_idx = sk->col_idx.as<uint32_t>();
    I.lval = sk->log_values.as<double>();
    I.col_ptr = sk->col_ptr.as<long long>();
    I.row_idx = sk->row_idx.as<uint32_t>();
    I.lval_t = sk->log_values_t.as<double>();
    I.la = W.la.as<double>();
    I.lb = W.lb.as<double>();
    I.cov_row = sk->cov_row.as<unsigned char>();
    I.cov_col = sk->cov_col.as<unsigned char>();
    I.lu = sk->lu.as<double>();
    I.lv = sk->lv.as<double>();
    I.masked_rows0 = sk->cov_empty_rows;
    I.masked_cols0 = sk->cov_empty_cols;
    I.exponent = exponents[k];
  }
  std::vector<BatchStatus> status_host(count, BatchStatus{});
  BatchArgs A{};
  A.max_iter = cfg.max_iter;
  A.delta = cfg.delta;
  A.policy = policy;
  A.npad = npad;
  const size_t smem = sizeof(double) * 2 * npad + sizeof(unsigned int) * 2 * (npad / 32);
  // fp32 sketches take the fp32-accurate exp (as spk_sketch_solve); a batch
  // mixing storage types runs its fp64 ones with fp64 exp in a second launch
  Timer tm(s);
  for (int f32 = 0; f32 < 2; ++f32) {
    std::vector<int> sel;
    for (int k = 0; k < count; ++k)
      if ((sks[k]->value_type == SPK_VALUES_F32 && !ctx->deterministic) == (f32 == 1)) sel.push_back(k);
    if (sel.empty() || cfg.max_iter <= 0) continue;
    DBuf d_sel_items;
    std::vector<BatchItem> part(sel.size());
    for (size_t q = 0; q < sel.size(); ++q) part[q] = items[sel[q]];
    upload(ctx, d_sel_items, part.data(), sizeof(BatchItem) * part.size());
    BatchArgs B = A;
    B.items = d_sel_items.as<BatchItem>();
    DBuf d_part_status(sizeof(BatchStatus) * sel.size());
    B.status = d_part_status.as<BatchStatus>();
    auto kern = f32 ? batch_log_kernel<LogKf> : batch_log_kernel<LogK>;
    loopcore::allow_max_dyn_smem((const void*)kern);
    kern<<<(int)sel.size(), kBatchThreads, smem, s>>>(B);
    ++ctx->launches;
    SPK_CUDA(cudaGetLastError());
    std::vector<BatchStatus> ps(sel.size());
    download(ctx, ps.data(), d_part_status, sizeof(BatchStatus) * sel.size());
    for (size_t q = 0; q < sel.size(); ++q) status_host[sel[q]] = ps[q];
  }
  const double secs = tm.stop();
  SPK_CUDA(cudaGetLastError());
  const std::vector<BatchStatus>& st = status_host;
  outs.assign(count, LoopOut{});
  errors.assign(count, std::string());
  error_kinds.assign(count, 0);
  for (int k = 0; k < count; ++k) {
    spk_sketch* sk = sks[k];
    const int64_t n = sk->n;
    LoopOut& o = outs[k];
    const BatchStatus& S = st[k];
    o.iterations = cfg.max_iter > 0 ? S.iterations : 0;
    o.converged = S.converged;
    o.masked_rows = cfg.max_iter > 0 ? S.masked_rows : sk->cov_empty_rows;
    o.masked_cols = cfg.max_iter > 0 ? S.masked_cols : sk->cov_empty_cols;
    o.loop_s = secs / std::max(count, 1);  // the batch's loop time, shared out
    if (S.error_kind == SPK_E_ZERO_DENOMINATOR) {
      error_kinds[k] = SPK_E_ZERO_DENOMINATOR;
      errors[k] = S.error_half == 0 ? "Kv vanished at row " + std::to_string(S.error_index)
                                    : "K'u vanished at column " + std::to_string(S.error_index);
    } else if (S.error_kind == SPK_E_DEGENERATE_SKETCH_ERROR) {
      error_kinds[k] = SPK_E_DEGENERATE_SKETCH_ERROR;
      errors[k] = "masking removed every atom";
    }
    sk->u.ensure(sizeof(double) * n);
    sk->v.ensure(sizeof(double) * n);
    if (cfg.max_iter <= 0) {  // no iteration: the initial scalings
      loopcore::init_scalings_kernel<true><<<loopcore::simple_grid(ctx, n), 256, 0, s>>>(
          n, sk->cov_row.as<unsigned char>(), sk->cov_col.as<unsigned char>(), sk->lu.as<double>(),
          sk->lv.as<double>());
      ++ctx->launches;
    }
    exp_pair_kernel<<<loopcore::simple_grid(ctx, n), 256, 0, s>>>(n, sk->lu.as<double>(), sk->lv.as<double>(),
                                                                  sk->u.as<double>(), sk->v.as<double>());
    ++ctx->launches;
  }
  SPK_CUDA(cudaStreamSynchronize(s));
}

}  // namespace spk
