// batch.cu -- many small log-domain Sparse Sinkhorn solves at once (config 3:
// 496 WFR frame pairs of n = 12,544, each run by pairwise_wfr,
// proj/src/harness.cpp:349-406, one spar_sink_uot at a time).
//
// A cluster of CS CTAs (CS = 2 by default: two SMs) owns one sketch for its
// whole solve. Every CTA keeps BOTH log scalings (lu, lv: 2 n fp64 = 196 KB at
// n = 12,544) in its own shared memory, so the gathered x of a half is a
// shared-memory read and the only HBM traffic is the sketch stream. A half
// is split over the cluster's CTAs by entry count; each CTA writes the new
// values of its rows into its own copy and, through DSMEM, into its peers'
// copies; one cluster barrier per half publishes them. Residual partials,
// mask counts and the first failing atom are exchanged through DSMEM after
// the same barrier and combined in rank order, so every CTA takes the same
// stop / failure decision. Clusters are independent (no grid barrier). Two
// SMs per pair also evens out the waves: 496 pairs = 3.35 waves of 148 SMs
// one CTA per pair (4 waves run), 6.7 waves as CTA pairs (7 run).
//
// Entry stream: fp32 sketches (config 3) stream ONE u64 per entry -- log K~
// as an fp64 rounded to a 35-bit mantissa (relative error 2^-35, far below
// the fp32 rounding of K~ itself) with the byte offset of the gathered x
// (column / row index << 3) in the low 17 bits (n <= 16,384: the batch limit
// is ~14k). 8 bytes per entry,
// SURVEY 8(d)'s V + I. fp64 sketches stream u32 indices + fp64 log K~ (12 B).
//
// Semantics: detail::log_scaling_loop (include/sparsink/solvers.hpp:397-513):
// lu = f (log a - LSE_j(log K~ + lv)); a row whose LSE is -inf is masked
// (Mask) or raises ZeroDenominator (Error); the stop rule sums |d lu| + |d lv|
// over unmasked atoms for t >= 2; all rows or all columns masked raises
// DegenerateSketchError. The LSE is one online pass (running max, rescaled
// sum) over blocks of U entries per lane, with the fp32-accurate exp for fp32
// sketches (as spk_sketch_solve) and fp64 exp for fp64 sketches; the single-
// sketch path sums in another order, so results agree to rounding
// (tests/test_gpu_batch.py, tests/test_gpu_fullsize.py quantify it).
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
#ifndef SPK_BATCH_G
#define SPK_BATCH_G 8
#endif
constexpr int kG = SPK_BATCH_G;  // lanes per row (config 3 rows: ~94 entries)
constexpr int kRows = 32 / kG;

struct BatchItem {
  int64_t n;
  const long long* row_ptr;
  const uint32_t* col_idx;            // split stream (fp64 sketches)
  const double* lval;
  const unsigned long long* lpack;    // packed stream (fp32 sketches)
  const long long* col_ptr;
  const uint32_t* row_idx;
  const double* lval_t;
  const unsigned long long* lpack_t;
  const double* la;  // log a (-inf where a = 0)
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


// Packed entry: log K~ as fp64 with its low 17 bits replaced by the byte
// offset of the gathered x (index << 3, index < 2^14): a 35-bit mantissa
// (relative 3e-11, far below the fp32 rounding of K~ itself).
constexpr unsigned long long kPackLowMask = 0x1ffffull;
constexpr uint32_t kPackOffMask = 0x1fff8u;
constexpr int64_t kPackMaxN = 1 << 14;

// Entry stream of one half: packed u64 (PACKED) or u32 index + fp64 log K~.
template <bool PACKED>
struct Stream {
  const unsigned long long* pk;
  const uint32_t* idx;
  const double* lv;
  // running position in the stream (pointers, so loads take immediate offsets)
  struct Cursor {
    const unsigned long long* pk;
    const uint32_t* idx;
    const double* lv;
    // jo: byte offset of the gathered x (index * 8), l: log K~
    __device__ __forceinline__ void load(int off, uint32_t& jo, double& l) const {
      if constexpr (PACKED) {
        const unsigned long long w = __ldg(pk + off);
        jo = (uint32_t)w & kPackOffMask;
        l = __longlong_as_double((long long)(w & ~kPackLowMask));
      } else {
        jo = __ldg(idx + off) << 3;
        l = __ldg(lv + off);
      }
    }
    __device__ __forceinline__ void advance(int d) {
      if constexpr (PACKED) pk += d;
      else {
        idx += d;
        lv += d;
      }
    }
  };
  __device__ __forceinline__ Cursor cursor(long long p) const {
    if constexpr (PACKED) return Cursor{pk + p, nullptr, nullptr};
    else return Cursor{nullptr, idx + p, lv + p};
  }
  __device__ __forceinline__ void prefetch_l2(long long b, long long e, int gl) const {
    const long long nb = (e - b) * (PACKED ? 8 : 12);
    const long long lines = (nb + 127) >> 7;
    for (long long q = gl; q < lines + (PACKED ? 0 : 1); q += kG) {
      const char* a;
      if constexpr (PACKED) {
        a = reinterpret_cast<const char*>(pk + b) + (q << 7);
      } else {
        const long long li = ((e - b) * 4 + 127) >> 7;
        a = q < li ? reinterpret_cast<const char*>(idx + b) + (q << 7)
                   : reinterpret_cast<const char*>(lv + b) + ((q - li) << 7);
      }
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
  }
};

// exp(d), d <= 0 (or -inf): fp32 MUFU.EX2 on the fp64-formed exponent (FAST)
// or fp64 exp
template <bool FAST>
__device__ __forceinline__ typename std::conditional<FAST, float, double>::type lse_term(double d) {
  if constexpr (FAST) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__double2float_rn(d) * 1.44269504088896341f));
    return r;
  } else {
    return exp(d);
  }
}

__device__ __forceinline__ double* peer_ptr(double* p, unsigned rank) {
  double* q;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(q) : "l"(p), "r"(rank));
  return q;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// First output atom of cluster rank r's share of a half: rows split by entry
// count (binary search on the row pointer).
__device__ __forceinline__ int64_t split_point(const long long* ptr, int64_t n, int r, int CS) {
  if (r <= 0) return 0;
  if (r >= CS) return n;
  const long long target = (long long)((__ldg(ptr + n) * (double)r) / CS);
  int64_t lo = 0, hi = n;  // first i with ptr[i] >= target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(ptr + mid) < target) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// One half over output atoms [i_lo, i_hi): out[i] for every unmasked atom from
// the row/column [ptr[i], ptr[i+1]) against the shared vector x. Writes the
// new value into this CTA's copy and into the CS-1 peers' copies. Returns
// this thread's residual share; masks and the first failing atom go through
// shared counters. 8 lanes share a row (4 rows per warp); each lane keeps U
// independent entry loads in flight; the next row group's entries are
// prefetched into L2 while this one finishes.
template <int CS, int U, bool PACKED, bool FAST>
__device__ __forceinline__ double batch_half(int64_t i_lo, int64_t i_hi, const long long* __restrict__ ptr,
                                             Stream<PACKED> st, const double* __restrict__ w, const double* x,
                                             double* out, unsigned int* ne, double exponent, int policy,
                                             long long* masks, unsigned long long* bad, unsigned my_rank) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & (kG - 1);
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  double err = 0.0;
  int64_t i = i_lo + (int64_t)warp * kRows + (lane / kG);
  long long bn = 0, en = 0;
  if (i < i_hi) {
    bn = __ldg(ptr + i);
    en = __ldg(ptr + i + 1);
  }
  for (int64_t i0 = i_lo + (int64_t)warp * kRows; i0 < i_hi; i0 += (int64_t)nw * kRows) {
    i = i0 + (lane / kG);
    const bool live = i < i_hi && ((ne[i >> 5] >> (i & 31)) & 1u);  // masked rows keep -inf
    const long long b = live ? bn : 0, e = live ? en : 0;
    {
      const int64_t inext = i + (int64_t)nw * kRows;
      if (inext < i_hi) {
        bn = __ldg(ptr + inext);
        en = __ldg(ptr + inext + 1);
      }
    }
    // online log-sum-exp: running max m (fp64) and the sum of exp(t - m).
    // FAST (fp32 sketches): each term's exponent t - m is formed in fp64 (no
    // cancellation), then exp2 runs on MUFU.EX2 and the lane's sum is fp32 --
    // the fp32 bar of the stored K~; fp64 sketches keep fp64 exp and sums.
    // A -inf term (K~ = 0 or a masked column) contributes exp(-inf) = 0.
    using Acc = typename std::conditional<FAST, float, double>::type;
    double m = -CUDART_INF;
    Acc s = 0;
    // this lane's entries: b + gl, b + gl + kG, ... (nk of them); full blocks
    // of U loads at immediate offsets from a running cursor, then one partial
    // block (32-bit counts: no 64-bit index arithmetic per load)
    const int cnt = (int)(e - b);
    int left = cnt > gl ? (cnt - gl + kG - 1) / kG : 0;
    typename Stream<PACKED>::Cursor cur = st.cursor(b + gl);
    auto block = [&](int nload) {
      double t[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        uint32_t jo = 0;
        double l = -CUDART_INF;
        if (k < nload) cur.load(k * kG, jo, l);
        // l = -inf (K~ = 0, or padding) or x = -inf (masked column): exp -> 0
        t[k] = l + *reinterpret_cast<const double*>(reinterpret_cast<const char*>(x) + jo);
      }
      // block maximum by compare-and-select (terms are finite or -inf, never
      // NaN: no NaN-aware fmax sequence, and no conversions on the MUFU/XU
      // pipe, which the exp2s already load)
      double M = t[0];
#pragma unroll
      for (int k = 1; k < U; ++k) M = t[k] > M ? t[k] : M;
      if (M == -CUDART_INF) return;  // every term of the block is -inf
      if (M > m) {
        s = (m == -CUDART_INF) ? Acc(0) : s * lse_term<FAST>(m - M);
        m = M;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) s += lse_term<FAST>(t[k] - m);
    };
    for (; left >= U; left -= U) {
      block(U);
      cur.advance(U * kG);
    }
    if (left > 0) block(left);
#pragma unroll
    for (int o = kG / 2; o; o >>= 1) {
      const double m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const Acc s2 = __shfl_xor_sync(0xffffffffu, s, o);
      const double M = fmax(m, m2);
      if (M != -CUDART_INF)
        s = (m == -CUDART_INF ? Acc(0) : s * lse_term<FAST>(m - M)) +
            (m2 == -CUDART_INF ? Acc(0) : s2 * lse_term<FAST>(m2 - M));
      m = M;
    }
    {  // the next row group's entries into L2 while this one finishes
      const int64_t inext = i + (int64_t)nw * kRows;
      if (inext < i_hi && en > bn) st.prefetch_l2(bn, en, gl);
    }
    if (live && gl == 0) {
      // FAST: the sum is fp32-accurate, so is its log (MUFU.LG2, ~2^-22 absolute
      // for s in [1, 256]) -- 2 instructions instead of the ~40 of an fp64 log
      const double lse = m == -CUDART_INF ? -CUDART_INF
                                          : m + (FAST ? (double)(__log2f((float)s) * 0.693147180559945f)
                                                      : log((double)s));
      double nv;
      bool write = true;
      if (lse == -CUDART_INF) {
        if (policy == SPK_POLICY_MASK) {  // :440-446 (masked atoms leave the residual)
          atomicAnd(ne + (i >> 5), ~(1u << (i & 31)));
          nv = -CUDART_INF;
          atomicAdd(reinterpret_cast<unsigned long long*>(masks), 1ull);
        } else {
          atomicMin(bad, (unsigned long long)i);
          write = false;
        }
      } else {
        nv = exponent * (__ldg(w + i) - lse);  // :449
        err += fabs(nv - out[i]);
      }
      if (write) {
        out[i] = nv;
#pragma unroll
        for (int r = 1; r < CS; ++r) *peer_ptr(out + i, (my_rank + r) % CS) = nv;
      }
    }
  }
  return err;
}

// Fixed-order CTA sum (warp sums, then every thread over the warps in order).
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

template <int CS, int U, bool PACKED, bool FAST>
__global__ void __launch_bounds__(kBatchThreads, 1) batch_log_kernel(BatchArgs A) {
  extern __shared__ __align__(16) double smem[];
  const unsigned rank = CS > 1 ? cluster_rank() : 0u;
  const BatchItem& I = A.items[blockIdx.x / CS];
  const int64_t n = I.n;
  double* lu = smem;
  double* lv = smem + A.npad;
  unsigned int* neu = reinterpret_cast<unsigned int*>(lv + A.npad);
  unsigned int* nev = neu + (A.npad >> 5);
  __shared__ double scratch[32];
  __shared__ long long masks_sh[2];
  __shared__ unsigned long long bad_sh[2];
  __shared__ double xe[2][CS];  // per half: every CTA's partials, slot = its rank
  __shared__ long long xm[2][CS];
  __shared__ unsigned long long xb[2][CS];
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
  // this CTA's share of the rows (u-half) and of the columns (v-half)
  const int64_t r0 = split_point(I.row_ptr, n, (int)rank, CS), r1 = split_point(I.row_ptr, n, (int)rank + 1, CS);
  const int64_t c0 = split_point(I.col_ptr, n, (int)rank, CS), c1 = split_point(I.col_ptr, n, (int)rank + 1, CS);
  const Stream<PACKED> srow{I.lpack, I.col_idx, I.lval};
  const Stream<PACKED> scol{I.lpack_t, I.row_idx, I.lval_t};
  long long mr = I.masked_rows0, mc = I.masked_cols0;
  long long t = 0;
  int converged = 0, ekind = 0, ehalf = 0;
  long long eidx = 0;
  if (CS > 1) cluster_barrier();  // peers' shared memory initialised before any DSMEM write
  else __syncthreads();
  // the half's cluster-wide outcome: residual, new masks, first failing atom
  // (cta_sum has synchronised the CTA: masks_sh / bad_sh are final.) Lanes
  // r < CS of warp 0 push this CTA's partials into slot [rank] of CTA r's
  // exchange arrays before the barrier; after it, every CTA sums its local
  // slots in rank order (the same values everywhere).
  auto exchange = [&](int h, double e_cta, double& e_all, long long& m_all, unsigned long long& b_all) {
    if (threadIdx.x < CS) {
      const unsigned r = threadIdx.x;
      double* pe = (CS == 1 || r == rank) ? &xe[h][rank] : peer_ptr(&xe[h][rank], r);
      long long* pm = reinterpret_cast<long long*>(
          (CS == 1 || r == rank) ? (double*)&xm[h][rank] : peer_ptr((double*)&xm[h][rank], r));
      unsigned long long* pb = reinterpret_cast<unsigned long long*>(
          (CS == 1 || r == rank) ? (double*)&xb[h][rank] : peer_ptr((double*)&xb[h][rank], r));
      *pe = e_cta;
      *pm = masks_sh[h];
      *pb = bad_sh[h];
    }
    if (CS > 1) cluster_barrier();  // new values + partials visible cluster-wide
    else __syncthreads();
    e_all = 0.0;
    m_all = 0;
    b_all = ~0ull;
#pragma unroll
    for (int r = 0; r < CS; ++r) {
      e_all += xe[h][r];
      m_all += xm[h][r];
      b_all = min(b_all, xb[h][r]);
    }
  };
  while (t < A.max_iter) {
    ++t;
    __syncthreads();  // every thread has read last iteration's counters
    if (threadIdx.x == 0) {
      masks_sh[0] = masks_sh[1] = 0;
      bad_sh[0] = bad_sh[1] = ~0ull;
    }
    __syncthreads();
    // u-half: rows of K~ against lv (kernel_log_apply, solvers.cpp:96-116)
    double eu, ev;
    long long mu, mv;
    unsigned long long bu, bv;
    exchange(0,
             cta_sum(batch_half<CS, U, PACKED, FAST>(r0, r1, I.row_ptr, srow, I.la, lv, lu, neu, I.exponent, A.policy,
                                                     &masks_sh[0], &bad_sh[0], rank),
                     scratch),
             eu, mu, bu);
    if (bu != ~0ull) {
      ekind = SPK_E_ZERO_DENOMINATOR;
      ehalf = 0;
      eidx = (long long)bu;
      break;
    }
    // v-half: columns against the NEW lu (Gauss-Seidel, :451-463)
    exchange(1,
             cta_sum(batch_half<CS, U, PACKED, FAST>(c0, c1, I.col_ptr, scol, I.lb, lu, lv, nev, I.exponent, A.policy,
                                                     &masks_sh[1], &bad_sh[1], rank),
                     scratch),
             ev, mv, bv);
    if (bv != ~0ull) {
      ekind = SPK_E_ZERO_DENOMINATOR;
      ehalf = 1;
      eidx = (long long)bv;
      break;
    }
    mr += mu;
    mc += mv;
    if (mr == n || mc == n) {  // :465-466
      ekind = SPK_E_DEGENERATE_SKETCH_ERROR;
      break;
    }
    if (t >= 2 && eu + ev <= A.delta) {  // :468-480
      converged = 1;
      break;
    }
  }
  if (CS > 1) cluster_barrier();  // every DSMEM access of the solve is complete before any CTA leaves
  // every CTA holds the full vectors: each stores its own share
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) I.lu[i] = lu[i];
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) I.lv[i] = lv[i];
  if (threadIdx.x == 0 && rank == 0) {
    BatchStatus& S = A.status[blockIdx.x / CS];
    S.iterations = t;
    S.masked_rows = mr;
    S.masked_cols = mc;
    S.converged = converged;
    S.error_kind = ekind;
    S.error_half = ehalf;
    S.error_index = eidx;
  }
}

// Packed entry stream of an fp32 sketch: log K~ (fp64 log of the stored fp32
// value, rounded to a 35-bit mantissa; -inf stays -inf) | index << 3.
__global__ void pack_log_kernel(const float* __restrict__ v, const uint32_t* __restrict__ idx, int64_t m,
                                unsigned long long* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const double l = log((double)v[k]);
    unsigned long long b = (unsigned long long)__double_as_longlong(l);
    if (isfinite(l)) b += (kPackLowMask + 1) >> 1;  // round to nearest on the kept bits
    out[k] = (b & ~kPackLowMask) | ((unsigned long long)idx[k] << 3);
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

// The packed (log K~ | index) streams of an fp32 sketch, built once.
static void ensure_log_packed(spk_ctx* ctx, spk_sketch* sk) {
  if (sk->log_packed.p) return;
  const int64_t m = std::max<int64_t>(sk->nnz, 1);
  sk->log_packed.alloc(sizeof(unsigned long long) * m);
  sk->log_packed_t.alloc(sizeof(unsigned long long) * m);
  if (sk->nnz == 0) return;
  const int g = loopcore::simple_grid(ctx, sk->nnz);
  pack_log_kernel<<<g, 256, 0, ctx->stream>>>(sk->values.as<float>(), sk->col_idx.as<uint32_t>(), sk->nnz,
                                              sk->log_packed.as<unsigned long long>());
  pack_log_kernel<<<g, 256, 0, ctx->stream>>>(sk->values_t.as<float>(), sk->row_idx.as<uint32_t>(), sk->nnz,
                                              sk->log_packed_t.as<unsigned long long>());
  ctx->launches += 2;
}

template <int CS, int U, bool PACKED, bool FAST>
static void launch_batch(spk_ctx* ctx, const BatchArgs& B, int count, size_t smem) {
  auto kern = batch_log_kernel<CS, U, PACKED, FAST>;
  loopcore::allow_max_dyn_smem((const void*)kern);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)(count * CS));
  lc.blockDim = dim3(kBatchThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  BatchArgs a = B;
  void* args[] = {&a};
  SPK_CUDA(cudaLaunchKernelExC(&lc, (const void*)kern, args));
}

template <bool PACKED, bool FAST>
static void launch_batch_cs(spk_ctx* ctx, const BatchArgs& B, int count, size_t smem) {
  const int cs = ctx->batch_cluster;
  const int u = ctx->batch_unroll;
  if (cs == 1) {
    if (u == 8) launch_batch<1, 8, PACKED, FAST>(ctx, B, count, smem);
    else launch_batch<1, 4, PACKED, FAST>(ctx, B, count, smem);
  } else if (cs == 4) {
    if (u == 8) launch_batch<4, 8, PACKED, FAST>(ctx, B, count, smem);
    else launch_batch<4, 4, PACKED, FAST>(ctx, B, count, smem);
  } else {
    if (u == 8) launch_batch<2, 8, PACKED, FAST>(ctx, B, count, smem);
    else launch_batch<2, 4, PACKED, FAST>(ctx, B, count, smem);
  }
}

// The batched loop over sks[0..count); returns per-item loop outcomes.
void run_batch_log(spk_ctx* ctx, spk_sketch* const* sks, int count, const spk_solver_cfg& cfg,
                   const std::vector<double>& exponents, int policy, std::vector<LoopOut>& outs,
                   std::vector<std::string>& errors, std::vector<int>& error_kinds) {
  cudaStream_t s = ctx->stream;
  NvtxRange nr("spk:batch_loop");
  int64_t nmax = 0;
  for (int k = 0; k < count; ++k) nmax = std::max(nmax, sks[k]->n);
  const int npad = (int)((nmax + 31) / 32 * 32);
  std::vector<BatchItem> items(count);
  for (int k = 0; k < count; ++k) {
    spk_sketch* sk = sks[k];
    const int64_t n = sk->n;
    const bool packed = sk->value_type == SPK_VALUES_F32;
    if (packed && n > kPackMaxN) fail(SPK_E_LENGTH_MISMATCH, "batched loop: dimension above 16384");
    ensure_coverage(ctx, sk);
    if (packed) ensure_log_packed(ctx, sk);
    else ensure_log_values(ctx, sk);
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
    I = BatchItem{};
    I.n = n;
    I.row_ptr = sk->row_ptr.as<long long>();
    I.col_ptr = sk->col_ptr.as<long long>();
    if (packed) {
      I.lpack = sk->log_packed.as<unsigned long long>();
      I.lpack_t = sk->log_packed_t.as<unsigned long long>();
    } else {
      I.col_idx = sk->col_idx.as<uint32_t>();
      I.lval = sk->log_values.as<double>();
      I.row_idx = sk->row_idx.as<uint32_t>();
      I.lval_t = sk->log_values_t.as<double>();
    }
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
  // fp32 sketches: packed stream + fp32-accurate exp (as spk_sketch_solve);
  // fp64 sketches: u32 + fp64 stream, fp64 exp -- one launch per storage type
  Timer tm(s);
  for (int f32 = 0; f32 < 2; ++f32) {
    std::vector<int> sel;
    for (int k = 0; k < count; ++k)
      if ((sks[k]->value_type == SPK_VALUES_F32) == (f32 == 1)) sel.push_back(k);
    if (sel.empty() || cfg.max_iter <= 0) continue;
    DBuf d_sel_items;
    std::vector<BatchItem> part(sel.size());
    for (size_t q = 0; q < sel.size(); ++q) part[q] = items[sel[q]];
    upload(ctx, d_sel_items, part.data(), sizeof(BatchItem) * part.size());
    BatchArgs B = A;
    B.items = d_sel_items.as<BatchItem>();
    DBuf d_part_status(sizeof(BatchStatus) * sel.size());
    B.status = d_part_status.as<BatchStatus>();
    if (f32) launch_batch_cs<true, true>(ctx, B, (int)sel.size(), smem);
    else launch_batch_cs<false, false>(ctx, B, (int)sel.size(), smem);
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
