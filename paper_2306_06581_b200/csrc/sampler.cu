// sampler.cu -- fused cost -> kernel -> plan normaliser -> Poisson sketch
// (north-star items 1 and 2).
//
// Reference semantics (proj/src/sparsify.cpp):
//   plans             ot_probabilities :71-91, uot_probabilities :93-115,
//                     uniform_probabilities :137-147, masked_grid_plan :49-67,
//                     shrink_with_uniform :149-167, SamplingPlan::prob
//                     (include/sparsink/sparsify.hpp:28-34)
//   sampling          poisson_sparsify :169-201 -- row i draws from
//                     CounterRng(seed, i); one draw per K_ij != 0 entry (also
//                     when p* <= 0); keep iff draw < p* = min(1, s p_ij);
//                     store p* >= 1 ? K_ij : K_ij / p*.
// The t-th draw of row i is splitmix64(mix_seed(seed,i) + t*golden)'s top 53
// bits (rng.hpp:24-40), and t = 1 + #(nonzero-K entries left of j in row i):
// a warp computes it with one ballot + popc per 32 columns, so rows are
// sampled in parallel with bit-identical index sets.
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "seqsum.h"
#include "internal.h"

namespace spk {

namespace {

// ---- kernel source --------------------------------------------------------------

struct KSrc {
  const double* K;  // dense (n*n) or nullptr
  const double* x;
  const double* y;
  int64_t n;
  int dim;
  int kind;
  double eta, scale, eps;
};

// K_ij exactly as kernel_from_cost(cost/scale, eps) (geometry.cpp:83-102).
__device__ __forceinline__ double kernel_entry(const KSrc& S, int64_t i, int64_t j) {
  if (S.K) return S.K[i * S.n + j];
  const double* p = S.x + i * S.dim;
  const double* q = S.y + j * S.dim;
  double c;
  if (S.kind == SPK_COST_SQEUCLID) c = cost_entry<0>(p, q, S.dim, S.eta);
  else if (S.kind == SPK_COST_EUCLID) c = cost_entry<1>(p, q, S.dim, S.eta);
  else c = cost_entry<2>(p, q, S.dim, S.eta);
  c = c / S.scale;
  return isinf(c) ? 0.0 : exp_ref(-c / S.eps);
}

// ---- plan ---------------------------------------------------------------------

struct DPlan {
  const double* row_w;
  const double* col_w;
  int kind;
  int factorized;
  double inv;
  double g_k;
  int theta_mode;  // 0 none, 1 lazy (factorized, prob()), 2 folded into the grid
  double omt;      // 1 - theta
  double unif;     // theta / kernel_nnz
};

// Grid entry before normalisation (what the reference stores in the n x n
// grid on the support): OT/barycenter ra_i*cb_j, UOT (pa_i*pb_j)*K^g_k,
// uniform 1.
__device__ __forceinline__ double grid_raw(const DPlan& P, int64_t i, int64_t j, double k) {
  if (P.kind == SPK_PLAN_UOT) return dmul(dmul(P.row_w[i], P.col_w[j]), pow(k, P.g_k));
  if (P.kind == SPK_PLAN_UNIFORM) return 1.0;
  return dmul(P.row_w[i], P.col_w[j]);
}

// SamplingPlan::prob(i, j) for a supported entry.
__device__ __forceinline__ double plan_prob(const DPlan& P, int64_t i, int64_t j, double k) {
  double base = P.factorized ? dmul(P.row_w[i], P.col_w[j]) : dmul(grid_raw(P, i, j, k), P.inv);
  if (P.theta_mode == 1) return base == 0.0 ? 0.0 : dadd(dmul(P.omt, base), P.unif);
  if (P.theta_mode == 2) return base > 0.0 ? dadd(dmul(P.omt, base), P.unif) : base;
  return base;
}

// ---- pass 0: c0 = max finite cost (geometry.cpp:61) --------------------------------

__global__ void max_cost_kernel(KSrc S, unsigned long long* out) {
  const int64_t total = S.n * S.n;
  double m = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / S.n, j = e - i * S.n;
    const double* p = S.x + i * S.dim;
    const double* q = S.y + j * S.dim;
    double c;
    if (S.kind == SPK_COST_SQEUCLID) c = cost_entry<0>(p, q, S.dim, S.eta);
    else if (S.kind == SPK_COST_EUCLID) c = cost_entry<1>(p, q, S.dim, S.eta);
    else c = cost_entry<2>(p, q, S.dim, S.eta);
    if (isfinite(c) && c > m) m = c;
  }
  m = warp_max(m);
  __shared__ double sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sm[w]);
    // non-negative doubles order like their bit patterns
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
  }
}

// The same maximum for the squared-Euclidean cost, tiled: a thread keeps its
// row's point in registers and walks a column range whose points are staged
// in shared memory (every lane reads the same y_j: a broadcast), four columns
// at a time. The per-pair kernel above spends its time on a 64-bit division
// and two point loads per pair (10.9 ms at n = 5e4, a third of config 5's
// end-to-end solve). d2 is formed exactly as cost_entry<0>: sequential over
// the dimensions, no FMA.
constexpr int kMaxTileJ = 512;
template <int DIM>
__global__ void __launch_bounds__(256) max_sqdist_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                         int64_t n, int col_parts, unsigned long long* out) {
  __shared__ double ys[kMaxTileJ * DIM];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (n + col_parts - 1) / col_parts;
  const int64_t j_lo = (int64_t)blockIdx.y * per, j_hi = min(n, j_lo + per);
  double xi[DIM];
#pragma unroll
  for (int k = 0; k < DIM; ++k) xi[k] = i < n ? x[i * DIM + k] : 0.0;
  double m = 0.0;
  for (int64_t j0 = j_lo; j0 < j_hi; j0 += kMaxTileJ) {
    const int cnt = (int)min((int64_t)kMaxTileJ, j_hi - j0);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * DIM; e += blockDim.x) ys[e] = y[j0 * DIM + e];
    __syncthreads();
    if (i < n) {
#pragma unroll 4
      for (int jj = 0; jj < cnt; ++jj) {
        double d2 = 0.0;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
          const double diff = dsub(xi[k], ys[jj * DIM + k]);
          d2 = dadd(d2, dmul(diff, diff));
        }
        if (d2 > m && isfinite(d2)) m = d2;
      }
    }
  }
  m = warp_max(m);
  __shared__ double sm[8];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = fmax(m, sm[w]);
    atomicMax(out, (unsigned long long)__double_as_longlong(m));  // non-negative doubles order like their bits
  }
}

// ---- pass 1: support count + grid row sums (masked_grid_plan :49-67) ------------

__global__ void plan_rows_kernel(KSrc S, DPlan P, long long* row_nnz, double* row_sum) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < S.n; i += nwarps) {
    long long cnt = 0;
    double acc = 0.0;
    for (int64_t j = lane; j < S.n; j += 32) {
      const double k = kernel_entry(S, i, j);
      if (k > 0.0) {
        ++cnt;
        acc += grid_raw(P, i, j, k);
      }
    }
    cnt = warp_sum_ll(cnt);
    acc = warp_sum(acc);
    if (lane == 0) {
      row_nnz[i] = cnt;
      row_sum[i] = acc;
    }
  }
}

// Deterministic single-block reduction of n row values (fixed order).
template <class T>
__global__ void reduce_rows_kernel(const T* v, int64_t n, T* out) {
  __shared__ T sm[1024];
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * per;
  const int64_t e = b + per < n ? b + per : n;
  T acc = 0;
  for (int64_t k = b; k < e; ++k) acc += v[k];
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

// ---- passes 2/3: Poisson sampling (poisson_sparsify :169-201) --------------------

template <bool EMIT, class VT>
__global__ void sample_rows_kernel(KSrc S, DPlan P, double s, uint64_t seed, int64_t row_base, int64_t n_rows,
                                   long long* row_cnt, const long long* row_ptr, uint32_t* col_out, VT* val_out) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t li = warp; li < n_rows; li += nwarps) {
    const int64_t i = row_base + li;  // global row: RNG stream, coordinates, plan weights
    const uint64_t state0 = mix_seed(seed, (uint64_t)i);
    uint64_t base_t = 0;
    long long cnt = 0;
    const long long out0 = EMIT ? row_ptr[li] : 0;
    for (int64_t j0 = 0; j0 < S.n; j0 += 32) {
      const int64_t j = j0 + lane;
      const double k = (j < S.n) ? kernel_entry(S, i, j) : 0.0;
      const bool nz = (k != 0.0);
      const unsigned m = __ballot_sync(0xffffffffu, nz);
      const uint64_t t = base_t + (uint64_t)__popc(m & lt_mask) + 1u;
      base_t += (uint64_t)__popc(m);
      bool keep = false;
      double ps = 0.0;
      if (nz) {
        ps = min1(dmul(s, plan_prob(P, i, j, k)));
        if (ps > 0.0) {
          if (ps >= 1.0) {
            keep = true;  // draw in [0, 1) is always below 1
          } else {
            const double draw = u64_to_unit(sm_finalize(state0 + t * kGolden));
            keep = draw < ps;
          }
        }
      }
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if (EMIT && keep) {
        const long long pos = out0 + cnt + __popc(km & lt_mask);
        col_out[pos] = (uint32_t)j;
        val_out[pos] = (VT)(ps >= 1.0 ? k : k / ps);
      }
      cnt += __popc(km);
    }
    if (!EMIT && lane == 0) row_cnt[li] = cnt;
  }
}

// ---- cached UOT kernel: K and K^g_k evaluated once for many (a, b) pairs ---------
// Same arithmetic and the same summation / draw order as plan_rows_kernel and
// sample_rows_kernel on the coordinate form (which the tiled kernels reproduce
// bit for bit), with the per-entry exp and pow replaced by two loads.

__global__ void cache_fill_kernel(KSrc S, double g_k, double* K, double* Kg) {
  const int64_t total = S.n * S.n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / S.n, j = e - i * S.n;
    const double k = kernel_entry(S, i, j);
    K[e] = k;
    Kg[e] = k != 0.0 ? pow(k, g_k) : 0.0;  // 0 < g_k < 1 and K <= 1: K^g_k >= K, so 0 marks the support exactly
  }
}

__global__ void plan_rows_cached_kernel(const double* Kg, int64_t n, DPlan P, long long* row_nnz, double* row_sum) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    long long cnt = 0;
    double acc = 0.0;
    const double rw = P.row_w[i];
    const double* row = Kg + i * n;
    for (int64_t j = lane; j < n; j += 32) {
      const double kg = __ldcs(row + j);
      if (kg != 0.0) {
        ++cnt;
        acc += dmul(dmul(rw, P.col_w[j]), kg);  // grid_raw (UOT)
      }
    }
    cnt = warp_sum_ll(cnt);
    acc = warp_sum(acc);
    if (lane == 0) {
      row_nnz[i] = cnt;
      row_sum[i] = acc;
    }
  }
}

// EMIT with slot_cap != nullptr: single pass into per-row slots (row_ptr = slot
// offsets; kept counts to row_cnt_i, a row outgrowing its slot sets *overflow
// and the caller redoes the sketch with the count / emit pair).
template <bool EMIT, class VT>
__global__ void sample_rows_cached_kernel(const double* K, const double* Kg, int64_t n, DPlan P, double s,
                                          uint64_t seed, long long* row_cnt, const long long* row_ptr,
                                          uint32_t* col_out, VT* val_out, const int* slot_cap = nullptr,
                                          int* row_cnt_i = nullptr, unsigned int* overflow = nullptr) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    const uint64_t state0 = mix_seed(seed, (uint64_t)i);
    const double rw = P.row_w[i];
    const double* row = Kg + i * n;
    uint64_t base_t = 0;
    long long cnt = 0;
    const long long out0 = EMIT ? row_ptr[i] : 0;
    for (int64_t j0 = 0; j0 < n; j0 += 32) {
      const int64_t j = j0 + lane;
      const double kg = (j < n) ? __ldcs(row + j) : 0.0;
      const bool nz = (kg != 0.0);
      const unsigned m = __ballot_sync(0xffffffffu, nz);
      const uint64_t t = base_t + (uint64_t)__popc(m & lt_mask) + 1u;
      base_t += (uint64_t)__popc(m);
      bool keep = false;
      double ps = 0.0;
      if (nz) {
        // plan_prob of a UOT grid entry: ((pa_i pb_j) K^g_k) inv, theta folded into the grid
        double base = dmul(dmul(dmul(rw, P.col_w[j]), kg), P.inv);
        if (P.theta_mode == 2) base = base > 0.0 ? dadd(dmul(P.omt, base), P.unif) : base;
        ps = min1(dmul(s, base));
        if (ps > 0.0) {
          if (ps >= 1.0) {
            keep = true;
          } else {
            const double draw = u64_to_unit(sm_finalize(state0 + t * kGolden));
            keep = draw < ps;
          }
        }
      }
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if (EMIT && keep) {
        const long long rel = cnt + __popc(km & lt_mask);
        if (!slot_cap || rel < slot_cap[i]) {
          const long long pos = out0 + rel;
          const double k = K[i * n + j];
          col_out[pos] = (uint32_t)j;
          val_out[pos] = (VT)(ps >= 1.0 ? k : k / ps);
        }
      }
      cnt += __popc(km);
    }
    if (!EMIT && lane == 0) row_cnt[i] = cnt;
    if (EMIT && slot_cap && lane == 0) {
      row_cnt_i[i] = (int)cnt;
      if (cnt > slot_cap[i]) atomicExch(overflow, 1u);
    }
  }
}

// ---- query helpers ------------------------------------------------------------

__global__ void plan_query_kernel(KSrc S, DPlan P, int64_t m, const int64_t* qi, const int64_t* qj,
                                  double* out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double k = kernel_entry(S, qi[q], qj[q]);
    out[q] = (k > 0.0) ? plan_prob(P, qi[q], qj[q], k) : (P.factorized ? plan_prob(P, qi[q], qj[q], k) : 0.0);
  }
}

__global__ void cost_query_kernel(KSrc S, int64_t m, const int64_t* qi, const int64_t* qj,
                                  double* cost, double* kern) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double* p = S.x + qi[q] * S.dim;
    const double* r = S.y + qj[q] * S.dim;
    double c;
    if (S.kind == SPK_COST_SQEUCLID) c = cost_entry<0>(p, r, S.dim, S.eta);
    else if (S.kind == SPK_COST_EUCLID) c = cost_entry<1>(p, r, S.dim, S.eta);
    else c = cost_entry<2>(p, r, S.dim, S.eta);
    c = c / S.scale;
    cost[q] = c;
    kern[q] = isinf(c) ? 0.0 : exp_ref(-c / S.eps);
  }
}

// ---- CSC mirror -----------------------------------------------------------------

__global__ void expand_rows_kernel(const long long* row_ptr, int64_t n, uint32_t* rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps)
    for (long long p = row_ptr[i] + lane; p < row_ptr[i + 1]; p += 32) rows[p] = (uint32_t)i;
}

__global__ void iota_kernel(uint32_t* v, int64_t m) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m;
       q += (int64_t)gridDim.x * blockDim.x)
    v[q] = (uint32_t)q;
}

__global__ void col_count_kernel(const uint32_t* col, int64_t m, long long* cnt) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m;
       q += (int64_t)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long*)&cnt[col[q]], 1ull);
}

template <class VT>
__global__ void gather_csc_kernel(const uint32_t* perm, const uint32_t* rows, const VT* vals,
                                  int64_t m, uint32_t* row_idx, VT* vals_t) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[q];
    row_idx[q] = rows[p];
    vals_t[q] = vals[p];
  }
}

template <class VT>
__global__ void sum_values_kernel(const VT* v, int64_t m, double* partial) {
  double acc = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m;
       q += (int64_t)gridDim.x * blockDim.x)
    acc += (double)v[q];
  acc = warp_sum(acc);
  __shared__ double sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sm[w];
    partial[blockIdx.x] = t;
  }
}

template <class VT>
__global__ void sum_values_seq_kernel(const VT* v, int64_t m, double* out) {
  double acc = 0.0;
  for (int64_t q = 0; q < m; ++q) acc = dadd(acc, (double)v[q]);
  *out = acc;
}

KSrc make_src(const DevKernel& dk) {
  KSrc S;
  S.K = dk.dense ? dk.K.as<double>() : nullptr;
  S.x = dk.x.as<double>();
  S.y = dk.y.as<double>();
  S.n = dk.n;
  S.dim = dk.dim;
  S.kind = dk.kind;
  S.eta = dk.eta;
  S.scale = dk.scale;
  S.eps = dk.eps;
  return S;
}

int grid_for_rows(spk_ctx* ctx, int64_t rows, int warps_per_block) {
  const int64_t need = (rows + warps_per_block - 1) / warps_per_block;
  const int64_t cap = (int64_t)ctx->num_sms * 16;
  return (int)std::max<int64_t>(1, std::min(need, cap));
}

int grid_for(spk_ctx* ctx, int64_t items, int threads) {
  const int64_t need = (items + threads - 1) / threads;
  const int64_t cap = (int64_t)ctx->num_sms * 32;
  return (int)std::max<int64_t>(1, std::min(need, cap));
}

// ==== tiled coordinate sampler (v3) ================================================
//
// One CTA = 8 warps x 4 rows; the CTA walks all columns in tiles of 256 points
// staged in shared memory (SoA, conflict-free), each warp handles 32 columns
// x its 4 rows per step, so every y_j is read from L2 once per 32 rows.
//
// Support (K_ij != 0  <=>  d2_ij < D0; D0 found once by a device bisection of
// the exact kernel_from_cost arithmetic, entries within 1e-12 of D0 take the
// exact path): screened first in fp32 -- d2 from fp32 copies of the points
// with an error bound 2^-18 (|x|^2 + |y|^2), far above the worst-case fp32
// error -- so the reference-order fp64 d2 is only computed for pairs the
// screen cannot decide.
//
// Draw: every supported entry consumes draw t of its row (t = 1 + #supported
// entries to its left: ballot + popc). keep needs u_t < p* <= P_i, a per-row
// bound of p*, so the screen evaluates only the top 32 bits of the splitmix64
// output (out_hi = z_hi ^ (z_hi >> 31), z_hi = mulhi of the last multiply)
// and rejects out_hi > floor(P_i 2^32) + 1; survivors (a ~P_i fraction)
// take the exact path: full draw, exact K (two IEEE divisions + exp), exact
// p* (SamplingPlan::prob), keep iff u < p*. Index sets are therefore the
// reference's bit for bit. Kept entries go straight into per-row slots sized
// from the plan pass (expected count + 6 sigma); a slot overflow falls back
// to the exact two-pass kernels above.
//
// Plan pass (masked_grid_plan): supported count per row and the row's grid
// mass -- for OT-like plans rw_i * (sum of all cb_j - sum of cb_j off the
// support), so supported pairs cost only the screen; UOT needs K^g_k on
// every supported pair and takes the exact path there.

#ifndef SPK_TILED_MINB
#define SPK_TILED_MINB 3  // resident CTAs per SM the tiled kernels are compiled for (80 registers)
#endif
#ifndef SPK_TILED_MINB_SCAN
// the OT-like sample pass is bound by the integer pipes, not by latency: 2 CTAs with 128 registers (no
// spills) measured 0.886 s against 0.898 s (3 CTAs) and 0.975 s (4) at config 4
#define SPK_TILED_MINB_SCAN 2
#endif
constexpr int kTileJ = 1024;
constexpr int kQueue = 160;  // candidate queue slots per warp: 31 left over + one step's 4 x 32
constexpr int kSuper = 8;  // column tiles tested at once for "every pair supported" (one scan over 8192 columns)
constexpr int kRPW = 4;  // rows per warp
constexpr int kTileRows = 8 * kRPW;

struct TiledArgs {
  const double* x;   // fp64 points (exact path)
  const double* y;
  const float* xf;   // fp32 copies and squared norms (screen)
  const float* yf;
  const float* xn;
  const float* yn;
  int64_t n;         // columns (target points)
  int64_t n_rows;    // rows handled (a slab of sources for sharded builds)
  int64_t row_base;  // global index of local row 0
  int dim, kind;
  double eta, scale, eps;
  double lo, hi;     // d2 < lo: supported; d2 >= hi: not; else exact
  float lof, hif;    // the same bounds in fp32 (rounded outwards)
  float mg;          // screen margin factor; +inf disables the screen
  const double* ytile_r;  // per column tile: max |y_j| (rounded up)
  const double* ysuper_r;  // per run of kSuper column tiles
  DPlan P;
  double s;
  uint64_t seed;
  double colw_total;  // plan pass: sum of all column weights
  double col_bound;   // sample pass: max column factor of the plan
  // plan mode
  long long* row_nnz;
  double* row_sum;
  // sample mode
  const long long* slot_off;
  const int* slot_cap;
  uint32_t* pool_col;
  void* pool_val;
  int* row_cnt;
  unsigned int* overflow;
};

__device__ __forceinline__ double exact_k(const TiledArgs& A, double d2) {
  return kernel_from_d2(A.kind, d2, A.eta, A.scale, A.eps);
}

// pairwise_cost's sequential d2 (geometry.cpp:16-59), no FMA.
template <int DIM>
__device__ __forceinline__ double exact_d2(const double* __restrict__ xp, const double* __restrict__ yp) {
  double d2 = 0.0;
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    const double diff = dsub(xp[k], yp[k]);
    d2 = dadd(d2, dmul(diff, diff));
  }
  return d2;
}

// Top 32 bits of sm_finalize(x) (the splitmix64 output): the last xor-shift
// only touches bit 0 of the high word, and the high word of the last product
// needs one mulhi and two low multiplies.
__device__ __forceinline__ uint32_t sm_finalize_hi(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = x ^ (x >> 27);
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  const uint32_t zh = __umulhi(lo, 0x133111ebu) + lo * 0x94d049bbu + hi * 0x133111ebu;
  return zh ^ (zh >> 31);
}

// Screen word of the fast scan: the high word zh of the last product, before
// the final xor-shift. out_hi = zh ^ (zh >> 31) differs from zh only when
// zh >= 2^31, and then both exceed any bound below 2^31; so for th < 2^31,
// out_hi <= th <=> zh <= th (rows with a larger bound use th2 = 2^32 - 1,
// i.e. always take the exact path).
// 17 integer instructions: the 64x64 product as one wide multiply plus two
// accumulating low multiplies (ptxas otherwise adds a fourth).
__device__ __forceinline__ uint32_t mulhi_pipe(uint32_t a, uint32_t b) {  // a * b >> 32 on the FMA pipe
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t sm_screen_hi(uint64_t x) {
  // one high-word right shift runs as IMAD.HI (FMA pipe): the hash is
  // otherwise ALU-pipe bound (shifts, xors, compares)
  uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  lo = lo ^ __funnelshift_r(lo, hi, 30);
  hi = hi ^ (hi >> 30);
  uint32_t plo, phi;
  asm("{\n\t.reg .u64 p;\n\t"
      "mul.wide.u32 p, %2, 0x1ce4e5b9;\n\t"
      "mov.b64 {%0, %1}, p;\n\t"
      "mad.lo.u32 %1, %2, 0xbf58476d, %1;\n\t"
      "mad.lo.u32 %1, %3, 0x1ce4e5b9, %1;\n\t}"
      : "=r"(plo), "=r"(phi)
      : "r"(lo), "r"(hi));
  // x ^ (x >> 27) on (phi:plo)
  lo = plo ^ __funnelshift_r(plo, phi, 27);
  hi = phi ^ (phi >> 27);  // (ALU: IMAD runs on the heavy FMA half only, measured 74% busy with both on it)
  return __umulhi(lo, 0x133111ebu) + lo * 0x94d049bbu + hi * 0x133111ebu;
}

// The grid entry / prob of a supported entry, given its row and column
// weights (same operations as grid_raw / plan_prob).
__device__ __forceinline__ double plan_prob_w(const DPlan& P, double rw, double cw, double k) {
  double base;
  if (P.factorized) {
    base = dmul(rw, cw);
  } else {
    const double g = (P.kind == SPK_PLAN_UOT) ? dmul(dmul(rw, cw), pow(k, P.g_k))
                     : (P.kind == SPK_PLAN_UNIFORM) ? 1.0 : dmul(rw, cw);
    base = dmul(g, P.inv);
  }
  if (P.theta_mode == 1) return base == 0.0 ? 0.0 : dadd(dmul(P.omt, base), P.unif);
  if (P.theta_mode == 2) return base > 0.0 ? dadd(dmul(P.omt, base), P.unif) : base;
  return base;
}

// Per-row screen threshold on out_hi: p* <= P_i for every supported j.
__device__ __forceinline__ uint32_t row_threshold(const TiledArgs& A, double rw) {
  const DPlan& P = A.P;
  double b;
  if (P.factorized) b = rw * A.col_bound;
  else b = ((P.kind == SPK_PLAN_UNIFORM) ? 1.0 : rw * A.col_bound) * P.inv;  // UOT: K^g_k <= 1
  if (P.theta_mode) b = P.omt * b + P.unif;
  const double Pi = A.s * b * (1.0 + 0x1p-30);
  if (!(Pi < 1.0)) return 0xffffffffu;
  const double t = floor(Pi * 4294967296.0) + 1.0;
  return t >= 4294967295.0 ? 0xffffffffu : (uint32_t)t;
}

// The exact decision of one screened entry (sparsify.cpp:188-197): K from the
// reference-order fp64 distance when not known yet, p* = min(1, s prob), keep
// iff the full draw falls below p*. Out of line: taken by a small fraction of
// entries, and inlined four times (one per row) it overflows the instruction
// cache (ncu: "no instruction" stalls dominated the UOT sample pass).
template <int DIM>
__device__ __noinline__ bool exact_keep(const TiledArgs& A, const double* xp, int64_t j, double rw, double cw,
                                        uint64_t x0, double& kv, double& ps) {
  if (kv < 0.0) kv = exact_k(A, exact_d2<DIM>(xp, A.y + j * DIM));
  ps = min1(dmul(A.s, plan_prob_w(A.P, rw, cw, kv)));
  return ps > 0.0 && (ps >= 1.0 || u64_to_unit(sm_finalize(x0)) < ps);
}

// Upper bound of K^g_k (UOT plan exponent) at squared distance >= d2lo, in
// fp32 with a 1e-4 relative slack (>> fp32 cos/log/exp error): K^g is
// decreasing in the distance, so the bound is evaluated at d2lo.
__device__ __forceinline__ double kg_upper(const TiledArgs& A, float d2lo) {
  const double gk = A.P.g_k;
  if (!(d2lo > 0.f) || gk <= 0.0) return 1.0;
  const float coef = (float)(gk / (A.scale * A.eps)) * (1.f - 1e-6f);  // rounded down
  float e;  // log2 of the bound
  if (A.kind == 0) {
    e = -coef * 1.44269504f * d2lo;
  } else if (A.kind == 1) {
    e = -coef * 1.44269504f * sqrtf(d2lo);
  } else {
    const float arg = sqrtf(d2lo) / (float)(2.0 * A.eta) * (1.f - 1e-6f);
    if (!(arg < 1.5707f)) return 1.0;  // at the support edge: no tightening
    // MUFU cos / lg2 / ex2: absolute error of __cosf ~4e-7 on [0, pi/2], so
    // the bound keeps its 1e-4 slack only where cos >= 0.01
    const float c = __cosf(arg);
    if (!(c >= 0.01f)) return 1.0;
    e = coef * __log2f(c * c);
  }
  return (double)exp2f(e) * (1.0 + 1e-4);
}

// Draw-screen threshold of one UOT entry: p* <= s (pa_i pb_j K^g_k) inv, with
// K^g_k bounded above (theta mixing as SamplingPlan::prob).
__device__ __forceinline__ uint32_t entry_threshold(const TiledArgs& A, double rw, double cw, float d2lo) {
  const DPlan& P = A.P;
  if (P.kind != SPK_PLAN_UOT) return 0xffffffffu;
  double b = rw * cw * kg_upper(A, d2lo) * P.inv;
  if (P.theta_mode) b = P.omt * b + P.unif;
  const double Pi = A.s * b * (1.0 + 0x1p-30);
  if (!(Pi < 1.0)) return 0xffffffffu;
  const double t = floor(Pi * 4294967296.0) + 1.0;
  return t >= 4294967295.0 ? 0xffffffffu : (uint32_t)t;
}

template <int DIM, bool SAMPLE, bool NEEDK, class VT>
__global__ void __launch_bounds__(256, (SAMPLE && !NEEDK) ? SPK_TILED_MINB_SCAN : SPK_TILED_MINB) tiled_kernel(TiledArgs A) {
  __shared__ float yfs[DIM][kTileJ];  // the screen's fp32 columns (exact paths read y from L2)
  __shared__ float yns[kTileJ];
  __shared__ double xmx[8];
  // Candidate queue (sample pass, all-supported tiles): a screened entry's
  // exact decision -- fp64 distance, two divisions, exp, the full draw -- runs
  // on ONE lane when taken where it is found (1.4% of the 128-pair steps at
  // config 4 hold a candidate), so candidates wait here, in row order, until
  // 32 of them fill a warp.
  // (static shared memory: the staged tile of DIM > 6 leaves no room for it)
  constexpr bool kUseQueue = SAMPLE && !NEEDK && DIM <= 6;
  constexpr int kQ = kUseQueue ? kQueue : 1;
  __shared__ uint32_t qj[8][kQ];   // column
  __shared__ uint32_t qt[8][kQ];   // draw index
  __shared__ unsigned char qr[8][kQ];  // row of the warp (0..3)
  __shared__ double q_rw[8][kRPW];
  __shared__ uint64_t q_st0[8][kRPW];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t groups = (A.n_rows + kTileRows - 1) / kTileRows;
  for (int64_t g = blockIdx.x; g < groups; g += gridDim.x) {
    float xr[kRPW][DIM];
    double xnorm[kRPW];  // |x_i| rounded up (inf for padding rows): whole-tile support test
    float xmg[kRPW];  // screen margin share of the row
    float d2s[kRPW];
    bool rvalid[kRPW];
    double rw[kRPW];
    uint64_t st0[kRPW];
    uint32_t th[kRPW];
    uint32_t th2[kRPW];  // fast-scan bound on zh (see sm_screen_hi)
    uint64_t lb[kRPW];   // stream base of the lane's draw: st0 + (lane + 1) * golden
    uint32_t tcnt[kRPW], cnt[kRPW];
    double racc[kRPW];
    int64_t row[kRPW];
    long long base[kRPW];
    int cap[kRPW];
#pragma unroll
    for (int q = 0; q < kRPW; ++q) {
      row[q] = g * kTileRows + w * kRPW + q;
      const bool valid = row[q] < A.n_rows;
      const int64_t gi = A.row_base + (valid ? row[q] : 0);
#pragma unroll
      for (int k = 0; k < DIM; ++k) xr[q][k] = valid ? A.xf[gi * DIM + k] : 0.f;
      xmg[q] = A.mg * (valid ? A.xn[gi] : 0.f);
      {
        double sq = 0.0;
#pragma unroll
        for (int k = 0; k < DIM; ++k) sq += A.x[gi * DIM + k] * A.x[gi * DIM + k];
        xnorm[q] = valid ? sqrt(sq) * (1.0 + 1e-15) : CUDART_INF;
      }
      rvalid[q] = valid;
      rw[q] = valid ? A.P.row_w[gi] : 0.0;
      st0[q] = mix_seed(A.seed, (uint64_t)gi);
      th[q] = SAMPLE ? row_threshold(A, rw[q]) : 0u;
      th2[q] = th[q] < 0x80000000u ? th[q] : 0xffffffffu;
      lb[q] = st0[q] + (uint64_t)(lane + 1) * kGolden;
      tcnt[q] = 0;
      cnt[q] = 0;
      racc[q] = 0.0;
      base[q] = (SAMPLE && valid) ? A.slot_off[row[q]] : 0;
      cap[q] = (SAMPLE && valid) ? A.slot_cap[row[q]] : 0;
    }
    int qn = 0;  // queued candidates (warp-uniform)
    if (kUseQueue) {
      __syncwarp();
      if (lane < kRPW) {
#pragma unroll
        for (int q = 0; q < kRPW; ++q)
          if (lane == q) {
            q_rw[w][q] = rw[q];
            q_st0[w][q] = st0[q];
          }
      }
      __syncwarp();
    }
    // Exact decisions of the first min(32, qn) queued candidates, one per lane
    // (same arithmetic and the same per-row output order as taking them in place).
    auto flush = [&]() {
      const int np = min(qn, 32);
      bool keep = false;
      double kv = -1.0, ps = 0.0;
      int myq = -1;
      uint32_t j = 0;
      if (lane < np) {
        myq = qr[w][lane];
        j = qj[w][lane];
        const uint64_t x0 = q_st0[w][myq] + (uint64_t)qt[w][lane] * kGolden;
        const double* xp = A.x + (A.row_base + g * kTileRows + w * kRPW + myq) * DIM;
        keep = exact_keep<DIM>(A, xp, (int64_t)j, q_rw[w][myq], A.P.col_w[j], x0, kv, ps);
      }
#pragma unroll
      for (int q = 0; q < kRPW; ++q) {
        const unsigned km = __ballot_sync(0xffffffffu, keep && myq == q);
        if (keep && myq == q) {
          const uint32_t pos = cnt[q] + (uint32_t)__popc(km & lt_mask);
          if (pos < (uint32_t)cap[q]) {
            A.pool_col[base[q] + pos] = j;
            static_cast<VT*>(A.pool_val)[base[q] + pos] = (VT)(ps >= 1.0 ? kv : kv / ps);
          }
        }
        cnt[q] += (uint32_t)__popc(km);
      }
      // the rest moves to the front
      __syncwarp();
      for (int b = 32; b < qn; b += 32) {
        const int e = b + lane;
        uint32_t tj = 0, tt = 0;
        unsigned char tr = 0;
        if (e < qn) {
          tj = qj[w][e];
          tt = qt[w][e];
          tr = qr[w][e];
        }
        __syncwarp();
        if (e < qn) {
          qj[w][e - 32] = tj;
          qt[w][e - 32] = tt;
          qr[w][e - 32] = tr;
        }
        __syncwarp();
      }
      qn -= np;
    };
    // largest |x_i| of the CTA's 32 rows (inf if any row is padding)
    double xmax_cta;
    {
      double m = xnorm[0];
#pragma unroll
      for (int q = 1; q < kRPW; ++q) m = fmax(m, xnorm[q]);
      __syncthreads();  // the previous group's readers of xmx are done
      if (lane == 0) xmx[w] = m;
      __syncthreads();
      xmax_cta = xmx[0];
#pragma unroll
      for (int k = 1; k < 8; ++k) xmax_cta = fmax(xmax_cta, xmx[k]);
    }
    int span = kTileJ;
    for (int64_t j0 = 0; j0 < A.n; j0 += span) {
      // |x_i - y_j| <= |x_i| + max_tile |y_j|: when that bound is inside the
      // support, every pair of the tile is supported. When it holds for all
      // 32 rows of the CTA no path reads the staged fp32 tile (the screen is
      // skipped; exact paths read y from L2), so the staging and both CTA
      // barriers are skipped too (every thread takes the same decision).
      // The same test on a run of kSuper tiles lets one scan cover all of
      // them (config 4: 99.9993% of the pairs are supported).
      span = kTileJ;
      double R;
      bool cta_all = false;
      if (j0 % ((int64_t)kTileJ * kSuper) == 0) {
        R = A.ysuper_r[j0 / ((int64_t)kTileJ * kSuper)];
        cta_all = (xmax_cta + R) * (xmax_cta + R) * (1.0 + 1e-12) < A.lo;
        if (cta_all) span = kTileJ * kSuper;
      }
      if (!cta_all) {
        R = A.ytile_r[j0 / kTileJ];
        cta_all = (xmax_cta + R) * (xmax_cta + R) * (1.0 + 1e-12) < A.lo;
      }
      if (!cta_all) {
        __syncthreads();
        for (int e = threadIdx.x; e < kTileJ * DIM; e += blockDim.x) {
          const int jj = e / DIM, k = e - jj * DIM;
          const int64_t j = j0 + jj;
          yfs[k][jj] = j < A.n ? A.yf[j * DIM + k] : 0.f;
        }
        for (int jj = threadIdx.x; jj < kTileJ; jj += blockDim.x) yns[jj] = j0 + jj < A.n ? A.yn[j0 + jj] : 0.f;
        __syncthreads();
      }
      const int jend = (int)min((int64_t)span, A.n - j0);
      bool tile_all = true;
#pragma unroll
      for (int q = 0; q < kRPW; ++q) {
        const double b = xnorm[q] + R;
        tile_all = tile_all && b * b * (1.0 + 1e-12) < A.lo;
      }
      if (!SAMPLE && !NEEDK && tile_all) continue;  // nothing off the support in this tile
      for (int c = 0; c < jend; c += 32) {
        if (SAMPLE && tile_all) {
          // every pair of the tile is supported: draw t of row q at lane l is
          // tcnt + l + 1. Scan 32-column steps with the 4 rows' screens
          // evaluated independently (no short-circuit: 4 hash chains in
          // flight per warp) until some lane may keep an entry.
          uint64_t xq[kRPW];  // draw input of the lane at tcnt (advanced by 64 golden per pass)
#pragma unroll
          for (int q = 0; q < kRPW; ++q) xq[q] = lb[q] + (uint64_t)tcnt[q] * kGolden;
          const int c_in = c;  // all four rows advance together: their draw counters follow c
          for (; c + 64 <= jend; c += 64) {  // two steps per pass: 8 independent chains
            bool c0 = false, c1 = false;
#pragma unroll
            for (int q = 0; q < kRPW; ++q) {
              c0 |= sm_screen_hi(xq[q]) <= th2[q];
              c1 |= sm_screen_hi(xq[q] + 32ull * kGolden) <= th2[q];
            }
            const bool a0 = __any_sync(0xffffffffu, c0), a1 = __any_sync(0xffffffffu, c1);
            if (a0 || a1) {
              if (!a0) c += 32;  // the first step keeps nothing: stop at the second
              break;
            }
#pragma unroll
            for (int q = 0; q < kRPW; ++q) xq[q] += 64ull * kGolden;
          }
#pragma unroll
          for (int q = 0; q < kRPW; ++q) tcnt[q] += (uint32_t)(c - c_in);
          for (; c + 32 <= jend; c += 32) {
            bool cand = false;
#pragma unroll
            for (int q = 0; q < kRPW; ++q) cand |= sm_screen_hi(lb[q] + (uint64_t)tcnt[q] * kGolden) <= th2[q];
            if (__any_sync(0xffffffffu, cand)) break;
#pragma unroll
            for (int q = 0; q < kRPW; ++q) tcnt[q] += 32u;
          }
          if (c >= jend) break;
          if (kUseQueue && c + 32 <= jend) {
            // a step that may keep something: queue the lanes whose exact
            // out_hi passes the row bound (draw t = tcnt + lane + 1: every
            // pair of the tile is supported)
#pragma unroll
            for (int q = 0; q < kRPW; ++q) {
              const uint32_t t = tcnt[q] + (uint32_t)lane + 1u;
              const bool cand = rvalid[q] && sm_finalize_hi(st0[q] + (uint64_t)t * kGolden) <= th[q];
              const unsigned m = __ballot_sync(0xffffffffu, cand);
              if (cand) {
                const int e = qn + __popc(m & lt_mask);
                qj[w][e] = (uint32_t)(j0 + c + lane);
                qt[w][e] = t;
                qr[w][e] = (unsigned char)q;
              }
              qn += __popc(m);
              tcnt[q] += 32u;
            }
            __syncwarp();
            while (qn >= 32) flush();
            continue;
          }
        }
        if (kUseQueue) {  // in-place decisions below write the same rows: queued ones go first
          while (qn > 0) flush();
        }
        const int jj = c + lane;
        const bool jvalid = jj < jend;
        const int64_t j = j0 + jj;
        const int js = jj & (kTileJ - 1);
        float yv[DIM];
#pragma unroll
        for (int k = 0; k < DIM; ++k) yv[k] = yfs[k][js];
        const float ymg = A.mg * yns[js];
        // fp32 screen of the 4 x 32 pairs (skipped when the tile is known supported)
        bool in[kRPW];
        bool all = true;
        if (tile_all) {
#pragma unroll
          for (int q = 0; q < kRPW; ++q) {
            in[q] = jvalid;
            d2s[q] = 0.f;
          }
          all = jvalid;
        } else {
#pragma unroll
          for (int q = 0; q < kRPW; ++q) {
            float d2f = 0.f;
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
              const float df = xr[q][k] - yv[k];
              d2f = fmaf(df, df, d2f);
            }
            in[q] = jvalid && rvalid[q] && d2f + (xmg[q] + ymg) < A.lof;
            all = all && in[q];
            d2s[q] = d2f;
          }
        }
        all = __all_sync(0xffffffffu, all);
        if (!SAMPLE && !NEEDK && all) continue;  // all on the support: nothing off it to count
        if (SAMPLE && all) {
          // every pair supported: draw t of row q at lane l is tcnt + l + 1
          bool cand = false;
#pragma unroll
          for (int q = 0; q < kRPW; ++q)
            cand = cand || sm_finalize_hi(st0[q] + (uint64_t)(tcnt[q] + lane + 1u) * kGolden) <= th[q];
          if (!__any_sync(0xffffffffu, cand)) {
#pragma unroll
            for (int q = 0; q < kRPW; ++q) tcnt[q] += 32u;
            continue;  // no draw can be below its p*: nothing kept in these 128 pairs
          }
        }
        // general path: exact classification where the screen could not tell
        const double cw = jvalid ? A.P.col_w[j] : 0.0;
#pragma unroll
        for (int q = 0; q < kRPW; ++q) {
          const bool valid = jvalid && rvalid[q];
          const double* xp = A.x + (A.row_base + row[q]) * DIM;
          double kv = -1.0;  // not computed
          bool nz;
          if (in[q]) {
            nz = true;
          } else if (!valid || d2s[q] - (xmg[q] + ymg) >= A.hif) {
            nz = false;
          } else {  // the screen cannot tell: reference arithmetic
            const double d2 = exact_d2<DIM>(xp, A.y + j * DIM);
            if (NEEDK || !(d2 < A.lo || d2 >= A.hi)) {
              kv = exact_k(A, d2);
              nz = kv != 0.0;
            } else {
              nz = d2 < A.lo;
            }
          }
          if (!SAMPLE) {
            if (NEEDK) {  // UOT grid (pa_i pb_j) K^g_k on every supported entry
              if (nz) {
                if (kv < 0.0) kv = exact_k(A, exact_d2<DIM>(xp, A.y + j * DIM));
                ++cnt[q];
                racc[q] += dmul(dmul(rw[q], cw), pow(kv, A.P.g_k));
              }
            } else if (valid && !nz) {  // off the support: count and weight
              ++cnt[q];
              racc[q] += cw;
            }
            continue;
          }
          const unsigned m = __ballot_sync(0xffffffffu, nz);
          const uint32_t t = tcnt[q] + (uint32_t)__popc(m & lt_mask) + 1u;
          tcnt[q] += (uint32_t)__popc(m);
          bool keep = false;
          double ps = 0.0;
          if (nz) {
            const uint64_t x0 = st0[q] + (uint64_t)t * kGolden;
            // UOT: the row bound assumes K^g_k <= 1 and the largest column
            // factor; this entry's own bound (its pb_j, K^g_k at a lower
            // bound of its distance) rejects most far entries before the
            // fp64 cost / exp / pow of the exact path
            // (no screen ran on an all-supported tile: its staged y, and so
            // ymg, may be stale -- no distance bound there)
            const float d2lo = tile_all ? 0.f : fmaxf(d2s[q] - (xmg[q] + ymg), 0.f);
            const uint32_t th_e = NEEDK ? min(th[q], entry_threshold(A, rw[q], cw, d2lo)) : th[q];
            if (sm_finalize_hi(x0) <= th_e)  // may be kept: exact draw, K and p* (out of line)
              keep = exact_keep<DIM>(A, xp, j, rw[q], cw, x0, kv, ps);
          }
          const unsigned km = __ballot_sync(0xffffffffu, keep);
          if (keep) {
            const uint32_t pos = cnt[q] + (uint32_t)__popc(km & lt_mask);
            if (pos < (uint32_t)cap[q]) {
              A.pool_col[base[q] + pos] = (uint32_t)j;
              static_cast<VT*>(A.pool_val)[base[q] + pos] = (VT)(ps >= 1.0 ? kv : kv / ps);
            }
          }
          cnt[q] += (uint32_t)__popc(km);
        }
      }
    }
    if (kUseQueue) {
      while (qn > 0) flush();
    }
#pragma unroll
    for (int q = 0; q < kRPW; ++q) {
      if (row[q] >= A.n_rows) continue;
      if (!SAMPLE) {
        const long long c = warp_sum_ll((long long)cnt[q]);
        const double sacc = warp_sum(racc[q]);
        if (lane == 0) {
          if (NEEDK) {
            A.row_nnz[row[q]] = c;
            A.row_sum[row[q]] = sacc;
          } else {  // c, sacc: count and column weight OFF the support
            const long long supp = A.n - c;
            A.row_nnz[row[q]] = supp;
            A.row_sum[row[q]] = (A.P.kind == SPK_PLAN_UNIFORM) ? (double)supp
                                                                : dmul(rw[q], dsub(A.colw_total, sacc));
          }
        }
      } else if (lane == 0) {
        A.row_cnt[row[q]] = (int)cnt[q];
        if ((int)cnt[q] > cap[q]) atomicExch(A.overflow, 1u);
      }
    }
  }
}

// smallest d2 with exact_k(d2) == 0 (bisection on the IEEE bit pattern)
__global__ void threshold_kernel(TiledArgs A, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  long long lo = 0;                                          // bits of +0.0
  long long hi = __double_as_longlong(CUDART_INF);           // K(inf) == 0
  if (exact_k(A, 0.0) == 0.0) {
    *out = 0.0;
    return;
  }
  while (hi - lo > 1) {
    const long long mid = lo + (hi - lo) / 2;
    if (exact_k(A, __longlong_as_double(mid)) > 0.0) lo = mid;
    else hi = mid;
  }
  *out = __longlong_as_double(hi);
}

// Largest |y_j| over each column tile, rounded up (whole-tile support test).
__global__ void tile_radius_kernel(const double* y, int64_t n, int dim, double* r) {
  const int64_t j0 = (int64_t)blockIdx.x * kTileJ;
  double m = 0.0;
  for (int64_t j = j0 + threadIdx.x; j < min(n, j0 + kTileJ); j += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < dim; ++k) s += y[j * dim + k] * y[j * dim + k];
    m = fmax(m, s);
  }
  m = warp_max(m);
  __shared__ double sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sm[w]);
    r[blockIdx.x] = isfinite(m) ? sqrt(m) * (1.0 + 1e-15) : CUDART_INF;
  }
}

__global__ void super_radius_kernel(const double* r, int64_t tiles, int64_t supers, double* rs) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= supers) return;
  double m = 0.0;
  for (int64_t t = s * kSuper; t < min(tiles, (s + 1) * kSuper); ++t) m = fmax(m, r[t]);
  rs[s] = m;
}

// fp32 copies of the points and their squared norms (screen inputs).
__global__ void to_f32_kernel(const double* x, int64_t n, int dim, float* xf, float* xn) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < dim; ++k) {
      const float v = (float)x[i * dim + k];
      xf[i * dim + k] = v;
      s += v * v;
    }
    xn[i] = s;
  }
}

// Upper bound of each row's expected kept count -> slot capacity
// (count is a sum of independent Bernoullis with mean <= U: cap U + 6 sqrt(U) + 16).
__global__ void slot_cap_kernel(int64_t n, int64_t row_base, int64_t n_cols, const long long* row_nnz,
                                const double* row_sum, const double* row_w, double col_w_total, int factorized,
                                double inv, double s, int theta_mode, double omt, double unif, int* cap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double supp = row_nnz ? (double)row_nnz[row_base + i] : (double)n_cols;
    double mass = factorized ? row_w[row_base + i] * col_w_total : row_sum[row_base + i] * inv;
    if (theta_mode) mass = omt * mass + unif * supp;
    const double u = fmin(supp, s * mass * (1.0 + 1e-9));
    const double c = fmin(supp, ceil(u + 6.0 * sqrt(u) + 16.0));
    cap[i] = (int)c;
  }
}

__global__ void compact_kernel(int64_t n, const long long* slot_off, const long long* row_ptr, const uint32_t* pool_col,
                               const unsigned char* pool_val, int vbytes, uint32_t* col, unsigned char* val) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    const long long src = slot_off[i], dst = row_ptr[i], m = row_ptr[i + 1] - row_ptr[i];
    for (long long k = lane; k < m; k += 32) {
      col[dst + k] = pool_col[src + k];
      if (vbytes == 4)
        reinterpret_cast<float*>(val)[dst + k] = reinterpret_cast<const float*>(pool_val)[src + k];
      else
        reinterpret_cast<double*>(val)[dst + k] = reinterpret_cast<const double*>(pool_val)[src + k];
    }
  }
}

__global__ void int_to_ll_kernel(const int* a, int64_t n, long long* b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <bool SAMPLE, bool NEEDK, class VT>
void launch_tiled(spk_ctx* ctx, const TiledArgs& A) {
  const int64_t groups = (A.n_rows + kTileRows - 1) / kTileRows;
  static const bool dbg = std::getenv("SPK_DEBUG_TIMING") != nullptr;
  std::unique_ptr<Timer> tm(dbg ? new Timer(ctx->stream) : nullptr);
#define SPK_TILED_CASE(D)                                                                                    \
  case D: {                                                                                                  \
    int occ = 0;                                                                                             \
    SPK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tiled_kernel<D, SAMPLE, NEEDK, VT>, 256, 0)); \
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(groups, (int64_t)ctx->num_sms * std::max(occ, 1))); \
    tiled_kernel<D, SAMPLE, NEEDK, VT><<<grid, 256, 0, ctx->stream>>>(A);                                    \
    break;                                                                                                   \
  }
  switch (A.dim) {
    SPK_TILED_CASE(1)
    SPK_TILED_CASE(2)
    SPK_TILED_CASE(3)
    SPK_TILED_CASE(4)
    SPK_TILED_CASE(5)
    SPK_TILED_CASE(6)
    SPK_TILED_CASE(8)
    SPK_TILED_CASE(10)
    default:
      fail(SPK_E_DIMENSION_MISMATCH, "tiled sampler: unsupported dimension");
  }
#undef SPK_TILED_CASE
  ++ctx->launches;
  SPK_CUDA(cudaGetLastError());
  if (tm) std::fprintf(stderr, "[timing] tiled_kernel<%s> %.4f s\n", SAMPLE ? "sample" : "plan", tm->stop());
}

bool tiled_dim_ok(int dim) { return dim == 1 || dim == 2 || dim == 3 || dim == 4 || dim == 5 || dim == 6 || dim == 8 || dim == 10; }

float f32_down(double v) {
  if (std::isinf(v)) return v > 0 ? INFINITY : -INFINITY;
  float f = (float)v;
  if ((double)f > v) f = std::nextafter(f, -INFINITY);
  return f;
}
float f32_up(double v) {
  if (std::isinf(v)) return v > 0 ? INFINITY : -INFINITY;
  float f = (float)v;
  if ((double)f < v) f = std::nextafter(f, INFINITY);
  return f;
}

TiledArgs tiled_args(spk_ctx* ctx, DevKernel& dk) {
  TiledArgs A{};
  const int64_t n = dk.n;
  if (!dk.xf.p) {
    dk.xf.alloc(sizeof(float) * n * dk.dim);
    dk.yf.alloc(sizeof(float) * n * dk.dim);
    dk.xn.alloc(sizeof(float) * n);
    dk.yn.alloc(sizeof(float) * n);
    to_f32_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(dk.x.as<double>(), n, dk.dim, dk.xf.as<float>(),
                                                                   dk.xn.as<float>());
    to_f32_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(dk.y.as<double>(), n, dk.dim, dk.yf.as<float>(),
                                                                   dk.yn.as<float>());
    const int64_t tiles = (n + kTileJ - 1) / kTileJ;
    const int64_t supers = (tiles + kSuper - 1) / kSuper;
    dk.ytr.alloc(sizeof(double) * (tiles + supers));  // tile radii, then the radii of runs of kSuper tiles
    tile_radius_kernel<<<(int)tiles, 256, 0, ctx->stream>>>(dk.y.as<double>(), n, dk.dim, dk.ytr.as<double>());
    super_radius_kernel<<<(int)((supers + 255) / 256), 256, 0, ctx->stream>>>(dk.ytr.as<double>(), tiles, supers,
                                                                               dk.ytr.as<double>() + tiles);
    ctx->launches += 4;
  }
  A.x = dk.x.as<double>();
  A.y = dk.y.as<double>();
  A.xf = dk.xf.as<float>();
  A.yf = dk.yf.as<float>();
  A.xn = dk.xn.as<float>();
  A.yn = dk.yn.as<float>();
  A.ytile_r = dk.ytr.as<double>();
  A.ysuper_r = dk.ytr.as<double>() + (n + kTileJ - 1) / kTileJ;
  A.n = n;
  A.n_rows = n;
  A.row_base = 0;
  A.dim = dk.dim;
  A.kind = dk.kind;
  A.eta = dk.eta;
  A.scale = dk.scale;
  A.eps = dk.eps;
  if (!dk.have_d0) {  // a property of the kernel (kind, eta, scale, eps): once per DevKernel
    DBuf d0(sizeof(double));
    threshold_kernel<<<1, 32, 0, ctx->stream>>>(A, d0.as<double>());
    ++ctx->launches;
    download(ctx, &dk.d0, d0, sizeof dk.d0);
    dk.have_d0 = true;
  }
  const double D0 = dk.d0;
  // exact-path band around the threshold (absorbs any non-monotone ULP effects)
  A.lo = D0 * (1.0 - 1e-12);
  A.hi = std::isinf(D0) ? D0 : D0 * (1.0 + 1e-12);
  A.lof = f32_down(A.lo);
  A.hif = f32_up(A.hi);
  // fp32 screen: |d2_f32 - d2| <= ~2^-20 (|x|^2 + |y|^2) for |coords| < 1e15;
  // 2^-18 leaves a 4x margin. Larger or non-finite coordinates: exact path only.
  A.mg = dk.max_abs < 1e15 ? 0x1p-18f : INFINITY;
  return A;
}

}  // namespace

// ---- host orchestration ----------------------------------------------------------

void make_dev_kernel(spk_ctx* ctx, const spk_kernel_desc* kd, double default_eps, DevKernel& dk,
                     bool need_cost) {
  if (!kd) fail(SPK_E_LENGTH_MISMATCH, "null kernel descriptor");
  const int64_t n = kd->n;
  if (n <= 0) fail(SPK_E_LENGTH_MISMATCH, "kernel dimension must be positive");
  dk.n = n;
  dk.eps = kd->kernel_epsilon > 0.0 ? kd->kernel_epsilon : default_eps;
  if (kd->K || (kd->C && !kd->x)) {
    dk.dense = true;
    dk.nnz_ratio = kd->nnz_ratio;
    if (kd->K) upload(ctx, dk.K, kd->K, sizeof(double) * n * n);  // cost-only form leaves K empty
    if (kd->C && need_cost) {
      upload(ctx, dk.C, kd->C, sizeof(double) * n * n);
      dk.have_cost = true;
    }
    return;
  }
  if (!kd->x || !kd->y || kd->dim <= 0)
    fail(SPK_E_DIMENSION_MISMATCH, "point lists must share a positive dimension");
  if (kd->cost_kind == SPK_COST_WFR && !(kd->eta > 0.0))
    fail(SPK_E_NON_POSITIVE_ETA, "eta = " + std::to_string(kd->eta));
  if (!(dk.eps > 0.0)) fail(SPK_E_NON_POSITIVE_EPSILON, "epsilon = " + std::to_string(dk.eps));
  dk.dense = false;
  dk.dim = kd->dim;
  dk.kind = kd->cost_kind;
  dk.eta = kd->eta;
  upload(ctx, dk.x, kd->x, sizeof(double) * n * kd->dim);
  upload(ctx, dk.y, kd->y, sizeof(double) * n * kd->dim);
  double mx = 0.0;  // any non-finite coordinate disables the fp32 screen
  for (int64_t k = 0; k < n * kd->dim; ++k) {
    const double ax = std::fabs(kd->x[k]), ay = std::fabs(kd->y[k]);
    mx = std::max(mx, std::isfinite(ax) ? ax : INFINITY);
    mx = std::max(mx, std::isfinite(ay) ? ay : INFINITY);
  }
  dk.max_abs = mx;
  dk.have_cost = true;
  if (kd->cost_scale > 0.0) {
    dk.scale = kd->cost_scale;
  } else {
    // c0 = max finite cost (geometry.cpp:61), the configs' max-normalisation.
    DBuf m(sizeof(unsigned long long));
    SPK_CUDA(cudaMemsetAsync(m.p, 0, m.bytes, ctx->stream));
    dk.scale = 1.0;
    KSrc S = make_src(dk);
    bool tiled = false;
    // cost = d2 itself (cost_entry<0>) or its correctly rounded square root (cost_entry<1>: monotone, so the
    // largest cost is the root of the largest d2)
    if ((dk.kind == SPK_COST_SQEUCLID || dk.kind == SPK_COST_EUCLID) && n >= 2048) {
      const int rb = (int)((n + 255) / 256);
      const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(64, (int64_t)ctx->num_sms * 8 / rb));
      const dim3 grid(rb, parts);
      tiled = true;
      switch (dk.dim) {
#define SPK_MAX_CASE(D)                                                                                      \
  case D:                                                                                                    \
    max_sqdist_kernel<D><<<grid, 256, 0, ctx->stream>>>(dk.x.as<double>(), dk.y.as<double>(), n, parts,      \
                                                        m.as<unsigned long long>());                         \
    break;
        SPK_MAX_CASE(1)
        SPK_MAX_CASE(2)
        SPK_MAX_CASE(3)
        SPK_MAX_CASE(4)
        SPK_MAX_CASE(5)
        SPK_MAX_CASE(6)
        SPK_MAX_CASE(8)
        SPK_MAX_CASE(10)
#undef SPK_MAX_CASE
        default: tiled = false;
      }
    }
    if (!tiled) max_cost_kernel<<<grid_for(ctx, n * n, 256), 256, 0, ctx->stream>>>(S, m.as<unsigned long long>());
    ++ctx->launches;
    unsigned long long bits = 0;
    SPK_CUDA(cudaMemcpyAsync(&bits, m.p, sizeof bits, cudaMemcpyDeviceToHost, ctx->stream));
    SPK_CUDA(cudaStreamSynchronize(ctx->stream));
    double c0;
    std::memcpy(&c0, &bits, sizeof c0);
    if (tiled && dk.kind == SPK_COST_EUCLID) c0 = std::sqrt(c0);
    dk.scale = c0;
    dk.max_normalised = true;
  }
}

namespace {
// Support fraction of a coordinate kernel from 4096 pseudo-random pairs.
__global__ void support_probe_kernel(KSrc S, unsigned int* hits) {
  const unsigned int t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t h = splitmix64(0x5eedull + t);
  const int64_t i = (int64_t)((h >> 32) % (uint64_t)S.n), j = (int64_t)((h & 0xffffffffull) % (uint64_t)S.n);
  const bool nz = kernel_entry(S, i, j) != 0.0;
  const unsigned m = __ballot_sync(0xffffffffu, nz);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(hits, (unsigned int)__popc(m));
}
}  // namespace

double probe_support_fraction(spk_ctx* ctx, DevKernel& dk) {
  if (dk.dense) return dk.nnz_ratio;
  DBuf hits(sizeof(unsigned int));
  SPK_CUDA(cudaMemsetAsync(hits.p, 0, sizeof(unsigned int), ctx->stream));
  KSrc S = make_src(dk);
  support_probe_kernel<<<16, 256, 0, ctx->stream>>>(S, hits.as<unsigned int>());
  ++ctx->launches;
  unsigned int h = 0;
  download(ctx, &h, hits, sizeof h);
  return (double)h / 4096.0;
}

bool cache_uot_kernel(spk_ctx* ctx, DevKernel& dk, double g_k) {
  if (dk.dense || !(g_k > 0.0 && g_k < 1.0)) return false;
  if (dk.cKg.p && dk.cache_g == g_k) return true;
  const int64_t n = dk.n;
  const double bytes = 16.0 * (double)n * (double)n;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return false;
  if (bytes > 8e9 || bytes > 0.4 * (double)free_b) return false;  // n <= ~22k, and never most of the free memory
  dk.cK.alloc(sizeof(double) * n * n);
  dk.cKg.alloc(sizeof(double) * n * n);
  KSrc S = make_src(dk);
  cache_fill_kernel<<<grid_for(ctx, n * n, 256), 256, 0, ctx->stream>>>(S, g_k, dk.cK.as<double>(),
                                                                         dk.cKg.as<double>());
  ++ctx->launches;
  SPK_CUDA(cudaGetLastError());
  dk.cache_g = g_k;
  return true;
}

bool plan_weights(spk_ctx* ctx, DevKernel& dk, const double* a, const double* b, int plan_kind, double lambda,
                  double eps, PlanInfo& plan) {
  const int64_t n = dk.n;
  plan.kind = plan_kind;
  plan.theta = 0.0;
  plan.g_k = 0.0;
  if (plan_kind == SPK_PLAN_UOT) {  // uot_probabilities argument checks (sparsify.cpp:96-97)
    if (!(lambda > 0.0)) fail(SPK_E_ERROR, "lambda must be > 0");
    if (!(eps > 0.0)) fail(SPK_E_NON_POSITIVE_EPSILON, "uot_probabilities");
  }
  // ---- host O(n) weights, in the reference's sequential order ----
  plan.row_w.assign(n, 0.0);
  plan.col_w.assign(n, 0.0);
  bool zero_mass = false;
  if (plan_kind == SPK_PLAN_OT) {  // sparsify.cpp:76-82
    double sa = 0.0, sb = 0.0;
    for (int64_t i = 0; i < n; ++i) sa += (plan.row_w[i] = std::sqrt(a[i]));
    for (int64_t j = 0; j < n; ++j) sb += (plan.col_w[j] = std::sqrt(b[j]));
    zero_mass = (sa == 0.0 || sb == 0.0);
    for (int64_t i = 0; i < n; ++i) plan.row_w[i] /= sa;
    for (int64_t j = 0; j < n; ++j) plan.col_w[j] /= sb;
  } else if (plan_kind == SPK_PLAN_UOT) {  // sparsify.cpp:102-107
    const double g_ab = lambda / (2.0 * lambda + eps);
    plan.g_k = eps / (2.0 * lambda + eps);
    auto powers = [&](const double* src, std::vector<double>& out) {
      WeightCache* wc = ctx->wcache;
      unsigned long long h = 1469598103934665603ull;
      if (wc) {
        for (int64_t i = 0; i < n; ++i) {
          unsigned long long bits;
          std::memcpy(&bits, src + i, sizeof bits);
          h = (h ^ bits) * 1099511628211ull;
        }
        for (const WeightCache::Entry& e : wc->entries)
          if (e.hash == h && e.exponent == g_ab && (int64_t)e.w.size() == n &&
              std::memcmp(e.src, src, sizeof(double) * n) == 0) {
            out = e.w;
            return;
          }
      }
      for (int64_t i = 0; i < n; ++i) out[i] = std::pow(src[i], g_ab);
      if (wc && wc->entries.size() < 256) wc->entries.push_back({src, h, g_ab, out});
    };
    powers(a, plan.row_w);
    powers(b, plan.col_w);
  } else if (plan_kind == SPK_PLAN_BARYCENTER) {  // sparsify.cpp:122-128
    double sb = 0.0;
    for (int64_t j = 0; j < n; ++j) sb += (plan.col_w[j] = std::sqrt(b[j]));
    zero_mass = (sb == 0.0);
    for (int64_t j = 0; j < n; ++j) plan.col_w[j] /= sb;
    for (int64_t i = 0; i < n; ++i) plan.row_w[i] = 1.0 / static_cast<double>(n);
  } else {  // uniform, sparsify.cpp:144
    for (int64_t i = 0; i < n; ++i) plan.row_w[i] = plan.col_w[i] = 1.0 / static_cast<double>(n);
  }

  plan.zero_mass = zero_mass;
  // ---- does the plan need the support / grid-normaliser pass over n^2 entries? ----
  const double nn = static_cast<double>(n) * static_cast<double>(n);
  bool need_pass = true;
  if (dk.dense) {
    // check_sizes (sparsify.cpp:41-46) on the given KernelMatrix::nnz_ratio
    if (std::llround(dk.nnz_ratio * nn) == 0) fail(SPK_E_ALL_ZERO_KERNEL, "kernel has no support");
    if (plan_kind != SPK_PLAN_UOT && dk.nnz_ratio == 1.0) need_pass = false;
  } else if (plan_kind != SPK_PLAN_UOT && dk.kind != SPK_COST_WFR && dk.max_normalised &&
             1.0 / dk.eps < 700.0) {
    // every C_ij = cost/c0 <= 1, so every K_ij >= exp(-1/eps) > 0: full support
    need_pass = false;
  }
  return need_pass;
}

void plan_pass_rows(spk_ctx* ctx, DevKernel& dk, const PlanInfo& plan, int64_t row0, int64_t row1,
                    long long* row_nnz, double* row_sum) {
  const int64_t n = dk.n;
  const int64_t rows = row1 - row0;
  if (rows <= 0) return;
  if (!plan.d_rw.p) {
    upload(ctx, plan.d_rw, plan.row_w.data(), sizeof(double) * n);
    upload(ctx, plan.d_cw, plan.col_w.data(), sizeof(double) * n);
  }
  DBuf &rw = plan.d_rw, &cw = plan.d_cw;
  DPlan P{};
  P.row_w = rw.as<double>();
  P.col_w = cw.as<double>();
  P.kind = plan.kind;
  P.g_k = plan.g_k;
  if (!dk.dense && plan.kind == SPK_PLAN_UOT && dk.cKg.p && dk.cache_g == plan.g_k && row0 == 0 && row1 == n) {
    plan_rows_cached_kernel<<<grid_for_rows(ctx, n, 8), 256, 0, ctx->stream>>>(dk.cKg.as<double>(), n, P, row_nnz,
                                                                                row_sum);
    ++ctx->launches;
  } else if (!dk.dense && tiled_dim_ok(dk.dim)) {
    TiledArgs A = tiled_args(ctx, dk);
    A.n_rows = rows;
    A.row_base = row0;
    A.P = P;
    A.row_nnz = row_nnz;
    A.row_sum = row_sum;
    double ct = 0.0;
    for (int64_t j = 0; j < n; ++j) ct += plan.col_w[j];
    A.colw_total = ct;
    if (plan.kind == SPK_PLAN_UOT) launch_tiled<false, true, double>(ctx, A);
    else launch_tiled<false, false, double>(ctx, A);
  } else {
    if (row0 != 0 || row1 != n) fail(SPK_E_DIMENSION_MISMATCH, "row-range plan pass needs the coordinate form");
    KSrc S = make_src(dk);
    plan_rows_kernel<<<grid_for_rows(ctx, n, 8), 256, 0, ctx->stream>>>(S, P, row_nnz, row_sum);
    ++ctx->launches;
  }
  // keep rw/cw alive until the pass has run (DBuf frees synchronously)
  SPK_CUDA(cudaStreamSynchronize(ctx->stream));
}

void plan_finish(spk_ctx* ctx, DevKernel& dk, bool need_pass, double theta, PlanInfo& plan) {
  const int64_t n = dk.n;
  const int plan_kind = plan.kind;
  const double nn = static_cast<double>(n) * static_cast<double>(n);
  long long support = static_cast<long long>(n) * n;
  double total = 0.0;
  if (need_pass) {
    // Fixed-order tree over the per-row sums: the same bits whichever GPU (or
    // set of GPUs) produced the rows.
    DBuf tot(sizeof(double)), tn(sizeof(long long));
    reduce_rows_kernel<double><<<1, 1024, 0, ctx->stream>>>(plan.d_row_sum.as<double>(), n, tot.as<double>());
    reduce_rows_kernel<long long><<<1, 1024, 0, ctx->stream>>>(plan.d_row_nnz.as<long long>(), n,
                                                               tn.as<long long>());
    ctx->launches += 2;
    SPK_CUDA(cudaMemcpyAsync(&total, tot.p, sizeof total, cudaMemcpyDeviceToHost, ctx->stream));
    SPK_CUDA(cudaMemcpyAsync(&support, tn.p, sizeof support, cudaMemcpyDeviceToHost, ctx->stream));
    SPK_CUDA(cudaStreamSynchronize(ctx->stream));
    // Equal grid terms (uniform marginals: config 4): the reference's
    // row-major sequential sum of the masked grid is a function of the support
    // count alone -- reproduce it bit for bit (seqsum.h). A tree sum differs
    // by 1.6e-5 relative at 10^12 terms (each sequential add drops the same
    // ulp fraction), which would move p* and flip sampled entries. Unequal
    // terms keep the tree (their sequential rounding errors are random, ~1e-12
    // relative at 10^8 terms: configs 2 and 3 show no index differences).
    if (plan_kind != SPK_PLAN_UOT && plan_kind != SPK_PLAN_UNIFORM && support > 0 &&
        std::all_of(plan.row_w.begin(), plan.row_w.end(), [&](double w) { return w == plan.row_w[0]; }) &&
        std::all_of(plan.col_w.begin(), plan.col_w.end(), [&](double w) { return w == plan.col_w[0]; }))
      total = seq_sum_const(plan.row_w[0] * plan.col_w[0], static_cast<uint64_t>(support));
  }
  const bool zero_mass = plan.zero_mass;
  if (!dk.dense) {
    dk.nnz_ratio = static_cast<double>(support) / nn;  // kernel_from_cost :100
    if (support == 0) fail(SPK_E_ALL_ZERO_KERNEL, "kernel has no support");
  }
  if (zero_mass) fail(SPK_E_ALL_ZERO_KERNEL, "zero-mass measure");

  plan.factorized = plan_kind != SPK_PLAN_UOT && dk.nnz_ratio == 1.0;
  if (plan.factorized) {
    plan.kernel_nnz = static_cast<int64_t>(n) * n;
    plan.inv = 1.0;
  } else {
    if (total <= 0.0) fail(SPK_E_ALL_ZERO_KERNEL, "no probability mass on support");
    plan.inv = 1.0 / total;  // masked_grid_plan multiplies by the reciprocal (:66-67)
    plan.kernel_nnz = support;
  }
  // shrink_with_uniform (sparsify.cpp:149-167); callers apply it for theta > 0
  if (theta != 0.0) {
    if (!(theta >= 0.0 && theta < 1.0)) fail(SPK_E_THETA_OUT_OF_RANGE, "theta = " + std::to_string(theta));
    plan.theta = theta;
  }
}

void build_plan(spk_ctx* ctx, DevKernel& dk, const double* a, const double* b, int plan_kind, double lambda,
                double eps, double theta, PlanInfo& plan) {
  const bool need_pass = plan_weights(ctx, dk, a, b, plan_kind, lambda, eps, plan);
  if (need_pass) {
    const int64_t n = dk.n;
    plan.d_row_nnz.alloc(sizeof(long long) * n);
    plan.d_row_sum.alloc(sizeof(double) * n);
    plan.have_rows = true;
    plan_pass_rows(ctx, dk, plan, 0, n, plan.d_row_nnz.as<long long>(), plan.d_row_sum.as<double>());
  }
  plan_finish(ctx, dk, need_pass, theta, plan);
}

namespace {

DPlan device_plan(const PlanInfo& plan, const double* rw, const double* cw) {
  DPlan P{};
  P.row_w = rw;
  P.col_w = cw;
  P.kind = plan.kind;
  P.factorized = plan.factorized ? 1 : 0;
  P.inv = plan.inv;
  P.g_k = plan.g_k;
  if (plan.theta > 0.0) {
    P.theta_mode = plan.factorized ? 1 : 2;
    P.omt = 1.0 - plan.theta;
    P.unif = plan.theta / static_cast<double>(plan.kernel_nnz);
  }
  return P;
}

}  // namespace

void plan_probs_query(spk_ctx* ctx, DevKernel& dk, const PlanInfo& plan, int64_t m,
                      const int64_t* qi, const int64_t* qj, double* out) {
  const int64_t n = dk.n;
  DBuf rw, cw, di, dj, dout(sizeof(double) * std::max<int64_t>(m, 1));
  upload(ctx, rw, plan.row_w.data(), sizeof(double) * n);
  upload(ctx, cw, plan.col_w.data(), sizeof(double) * n);
  upload(ctx, di, qi, sizeof(int64_t) * m);
  upload(ctx, dj, qj, sizeof(int64_t) * m);
  DPlan P = device_plan(plan, rw.as<double>(), cw.as<double>());
  KSrc S = make_src(dk);
  plan_query_kernel<<<grid_for(ctx, m, 256), 256, 0, ctx->stream>>>(S, P, m, di.as<int64_t>(),
                                                                     dj.as<int64_t>(), dout.as<double>());
  ++ctx->launches;
  download(ctx, out, dout, sizeof(double) * m);
}

namespace {
__global__ void kernel_from_cost_kernel(const double* C, int64_t m, double eps, double* K, unsigned long long* nnz) {
  unsigned long long local = 0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    const double c = C[q];
    const double v = isinf(c) ? 0.0 : exp_ref(-c / eps);  // geometry.cpp:95
    K[q] = v;
    local += v > 0.0 ? 1 : 0;
  }
  local = (unsigned long long)warp_sum_ll((long long)local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(nnz, local);
}
}  // namespace

void kernel_from_cost_dev(spk_ctx* ctx, const double* C_host, int64_t count, double eps, double* K_host,
                          int64_t* nnz) {
  if (!(eps > 0.0)) fail(SPK_E_NON_POSITIVE_EPSILON, "epsilon = " + std::to_string(eps));
  DBuf dc, dk(sizeof(double) * std::max<int64_t>(count, 1)), dn(sizeof(unsigned long long));
  upload(ctx, dc, C_host, sizeof(double) * count);
  SPK_CUDA(cudaMemsetAsync(dn.p, 0, dn.bytes, ctx->stream));
  kernel_from_cost_kernel<<<grid_for(ctx, count, 256), 256, 0, ctx->stream>>>(dc.as<double>(), count, eps,
                                                                              dk.as<double>(),
                                                                              dn.as<unsigned long long>());
  ++ctx->launches;
  download(ctx, K_host, dk, sizeof(double) * count);
  unsigned long long c = 0;
  download(ctx, &c, dn, sizeof c);
  if (nnz) *nnz = (int64_t)c;
}

void cost_kernel_query(spk_ctx* ctx, DevKernel& dk, int64_t m, const int64_t* qi, const int64_t* qj,
                       double* cost, double* kern) {
  DBuf di, dj, dc(sizeof(double) * std::max<int64_t>(m, 1)), dkk(sizeof(double) * std::max<int64_t>(m, 1));
  upload(ctx, di, qi, sizeof(int64_t) * m);
  upload(ctx, dj, qj, sizeof(int64_t) * m);
  KSrc S = make_src(dk);
  cost_query_kernel<<<grid_for(ctx, m, 256), 256, 0, ctx->stream>>>(S, m, di.as<int64_t>(), dj.as<int64_t>(),
                                                                    dc.as<double>(), dkk.as<double>());
  ++ctx->launches;
  if (cost) download(ctx, cost, dc, sizeof(double) * m);
  if (kern) download(ctx, kern, dkk, sizeof(double) * m);
}

void sample_sketch(spk_ctx* ctx, DevKernel& dk, const PlanInfo& plan, double s, uint64_t seed,
                   int value_type, spk_sketch* sk, int64_t row0, int64_t row1) {
  const int64_t ncols = dk.n;
  if (row1 < 0) row1 = ncols;
  const int64_t n = row1 - row0;  // rows sampled here (all of them unless sharded)
  const double nn = static_cast<double>(ncols) * static_cast<double>(ncols);
  if (!(s > 0.0) || s >= nn) fail(SPK_E_BUDGET_TOO_LARGE, "budget s must satisfy 0 < s < n^2");
  if (!plan.d_rw.p) {
    upload(ctx, plan.d_rw, plan.row_w.data(), sizeof(double) * ncols);
    upload(ctx, plan.d_cw, plan.col_w.data(), sizeof(double) * ncols);
  }
  DBuf &rw = plan.d_rw, &cw = plan.d_cw;
  DPlan P = device_plan(plan, rw.as<double>(), cw.as<double>());
  KSrc S = make_src(dk);

  sk->n = n;
  sk->n_cols = (n == ncols) ? 0 : ncols;
  sk->row_base = row0;
  sk->seed = seed;
  sk->value_type = value_type;
  sk->kernel_nnz = plan.kernel_nnz;
  sk->factorized_plan = plan.factorized ? 1 : 0;
  sk->plan_kind = plan.kind;
  sk->plan_inv = plan.inv;
  sk->plan_g_k = plan.g_k;
  sk->plan_theta = plan.theta;
  sk->row_ptr.alloc(sizeof(long long) * (n + 1));
  const size_t vbytes = value_type == SPK_VALUES_F32 ? 4 : 8;

  const bool cached = !dk.dense && plan.kind == SPK_PLAN_UOT && !plan.factorized && dk.cKg.p &&
                      dk.cache_g == plan.g_k && row0 == 0 && n == ncols;
  if (cached) {
    // ---- K and K^g_k of this kernel are resident (batched UOT sketches) ----
    const int grid = grid_for_rows(ctx, n, 8);
    if (plan.have_rows && !ctx->force_two_pass) {
      // single pass into row slots sized from the plan's row masses (as the tiled sampler)
      DBuf cap(sizeof(int) * n), capll(sizeof(long long) * n), off(sizeof(long long) * (n + 1));
      slot_cap_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(
          n, 0, dk.n, plan.d_row_nnz.as<long long>(), plan.d_row_sum.as<double>(), rw.as<double>(), 0.0, 0, plan.inv,
          s, P.theta_mode, P.omt, P.unif, cap.as<int>());
      int_to_ll_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(cap.as<int>(), n, capll.as<long long>());
      ctx->launches += 2;
      SPK_CUDA(cudaMemsetAsync(off.p, 0, sizeof(long long), ctx->stream));
      size_t tb = 0;
      SPK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, capll.as<long long>(), off.as<long long>() + 1, (int)n,
                                             ctx->stream));
      ctx->scratch.ensure(tb);
      SPK_CUDA(cub::DeviceScan::InclusiveSum(ctx->scratch.p, tb, capll.as<long long>(), off.as<long long>() + 1,
                                             (int)n, ctx->stream));
      long long pool = 0;
      SPK_CUDA(cudaMemcpyAsync(&pool, off.as<long long>() + n, sizeof pool, cudaMemcpyDeviceToHost, ctx->stream));
      SPK_CUDA(cudaStreamSynchronize(ctx->stream));
      DBuf &pcol = tmp_buf(ctx, 11, sizeof(uint32_t) * std::max<long long>(pool, 1)),
           &pval = tmp_buf(ctx, 12, vbytes * std::max<long long>(pool, 1));
      DBuf rcnt(sizeof(int) * n), ovf(sizeof(unsigned int));
      SPK_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(unsigned int), ctx->stream));
      if (value_type == SPK_VALUES_F32)
        sample_rows_cached_kernel<true, float><<<grid, 256, 0, ctx->stream>>>(
            dk.cK.as<double>(), dk.cKg.as<double>(), n, P, s, seed, nullptr, off.as<long long>(),
            pcol.as<uint32_t>(), pval.as<float>(), cap.as<int>(), rcnt.as<int>(), ovf.as<unsigned int>());
      else
        sample_rows_cached_kernel<true, double><<<grid, 256, 0, ctx->stream>>>(
            dk.cK.as<double>(), dk.cKg.as<double>(), n, P, s, seed, nullptr, off.as<long long>(),
            pcol.as<uint32_t>(), pval.as<double>(), cap.as<int>(), rcnt.as<int>(), ovf.as<unsigned int>());
      ++ctx->launches;
      unsigned int overflow = 0;
      download(ctx, &overflow, ovf, sizeof overflow);
      if (!overflow) {
        int_to_ll_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(rcnt.as<int>(), n, capll.as<long long>());
        ++ctx->launches;
        SPK_CUDA(cudaMemsetAsync(sk->row_ptr.p, 0, sizeof(long long), ctx->stream));
        SPK_CUDA(cub::DeviceScan::InclusiveSum(ctx->scratch.p, tb, capll.as<long long>(),
                                               sk->row_ptr.as<long long>() + 1, (int)n, ctx->stream));
        long long nnz = 0;
        SPK_CUDA(cudaMemcpyAsync(&nnz, sk->row_ptr.as<long long>() + n, sizeof nnz, cudaMemcpyDeviceToHost,
                                 ctx->stream));
        SPK_CUDA(cudaStreamSynchronize(ctx->stream));
        if (nnz > 0xffffffffLL) fail(SPK_E_BUDGET_TOO_LARGE, "sketch exceeds 2^32 entries");
        sk->nnz = nnz;
        sk->col_idx.alloc(sizeof(uint32_t) * std::max<long long>(nnz, 1));
        sk->values.alloc(vbytes * std::max<long long>(nnz, 1));
        compact_kernel<<<grid_for_rows(ctx, n, 8), 256, 0, ctx->stream>>>(
            n, off.as<long long>(), sk->row_ptr.as<long long>(), pcol.as<uint32_t>(), pval.as<unsigned char>(),
            (int)vbytes, sk->col_idx.as<uint32_t>(), sk->values.as<unsigned char>());
        ++ctx->launches;
        SPK_CUDA(cudaGetLastError());
        build_csc(ctx, sk);
        sk->kernel_mean = sketch_kernel_mean(ctx, sk);
        return;
      }
      // a row outgrew its slot: the exact count / emit pair below
    }
    DBuf cnt(sizeof(long long) * n);
    sample_rows_cached_kernel<false, double><<<grid, 256, 0, ctx->stream>>>(
        dk.cK.as<double>(), dk.cKg.as<double>(), n, P, s, seed, cnt.as<long long>(), nullptr, nullptr, nullptr);
    ++ctx->launches;
    SPK_CUDA(cudaMemsetAsync(sk->row_ptr.p, 0, sizeof(long long), ctx->stream));
    size_t tmp_bytes = 0;
    SPK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, cnt.as<long long>(), sk->row_ptr.as<long long>() + 1,
                                           (int)n, ctx->stream));
    ctx->scratch.ensure(tmp_bytes);
    SPK_CUDA(cub::DeviceScan::InclusiveSum(ctx->scratch.p, tmp_bytes, cnt.as<long long>(),
                                           sk->row_ptr.as<long long>() + 1, (int)n, ctx->stream));
    ++ctx->launches;
    long long nnz = 0;
    SPK_CUDA(cudaMemcpyAsync(&nnz, sk->row_ptr.as<long long>() + n, sizeof nnz, cudaMemcpyDeviceToHost,
                             ctx->stream));
    SPK_CUDA(cudaStreamSynchronize(ctx->stream));
    if (nnz > 0xffffffffLL) fail(SPK_E_BUDGET_TOO_LARGE, "sketch exceeds 2^32 entries");
    sk->nnz = nnz;
    sk->col_idx.alloc(sizeof(uint32_t) * std::max<long long>(nnz, 1));
    sk->values.alloc(vbytes * std::max<long long>(nnz, 1));
    if (value_type == SPK_VALUES_F32)
      sample_rows_cached_kernel<true, float><<<grid, 256, 0, ctx->stream>>>(
          dk.cK.as<double>(), dk.cKg.as<double>(), n, P, s, seed, nullptr, sk->row_ptr.as<long long>(),
          sk->col_idx.as<uint32_t>(), sk->values.as<float>());
    else
      sample_rows_cached_kernel<true, double><<<grid, 256, 0, ctx->stream>>>(
          dk.cK.as<double>(), dk.cKg.as<double>(), n, P, s, seed, nullptr, sk->row_ptr.as<long long>(),
          sk->col_idx.as<uint32_t>(), sk->values.as<double>());
    ++ctx->launches;
    SPK_CUDA(cudaGetLastError());
    build_csc(ctx, sk);
    sk->kernel_mean = sketch_kernel_mean(ctx, sk);
    return;
  }
  if (!dk.dense && tiled_dim_ok(dk.dim) && (plan.factorized || plan.have_rows) && !ctx->force_two_pass) {
    // ---- single pass: row slots sized from the plan's row masses ----
    DBuf cap(sizeof(int) * n), capll(sizeof(long long) * n), off(sizeof(long long) * (n + 1));
    double col_total = 0.0;
    for (int64_t j = 0; j < ncols; ++j) col_total += plan.col_w[j];
    slot_cap_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(
        n, row0, dk.n, plan.have_rows ? plan.d_row_nnz.as<long long>() : nullptr,
        plan.have_rows ? plan.d_row_sum.as<double>() : nullptr, rw.as<double>(), col_total,
        plan.factorized ? 1 : 0, plan.inv, s, P.theta_mode, P.omt, P.unif, cap.as<int>());
    int_to_ll_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(cap.as<int>(), n, capll.as<long long>());
    ctx->launches += 2;
    SPK_CUDA(cudaMemsetAsync(off.p, 0, sizeof(long long), ctx->stream));
    size_t tb = 0;
    SPK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, capll.as<long long>(), off.as<long long>() + 1, (int)n,
                                           ctx->stream));
    ctx->scratch.ensure(tb);
    SPK_CUDA(cub::DeviceScan::InclusiveSum(ctx->scratch.p, tb, capll.as<long long>(), off.as<long long>() + 1, (int)n,
                                           ctx->stream));
    long long pool = 0;
    SPK_CUDA(cudaMemcpyAsync(&pool, off.as<long long>() + n, sizeof pool, cudaMemcpyDeviceToHost, ctx->stream));
    SPK_CUDA(cudaStreamSynchronize(ctx->stream));
    DBuf &pcol = tmp_buf(ctx, 11, sizeof(uint32_t) * std::max<long long>(pool, 1)),
         &pval = tmp_buf(ctx, 12, vbytes * std::max<long long>(pool, 1));
    DBuf rcnt(sizeof(int) * n), ovf(sizeof(unsigned int));
    SPK_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(unsigned int), ctx->stream));
    TiledArgs A = tiled_args(ctx, dk);
    A.n_rows = n;
    A.row_base = row0;
    A.P = P;
    A.s = s;
    A.seed = seed;
    double cb = 0.0;  // largest column factor of the plan (UOT: pb_j; K^g_k <= 1)
    for (int64_t j = 0; j < ncols; ++j) cb = std::max(cb, plan.col_w[j]);
    A.col_bound = cb;
    A.slot_off = off.as<long long>();
    A.slot_cap = cap.as<int>();
    A.pool_col = pcol.as<uint32_t>();
    A.pool_val = pval.p;
    A.row_cnt = rcnt.as<int>();
    A.overflow = ovf.as<unsigned int>();
    const bool uotk = plan.kind == SPK_PLAN_UOT;
    if (value_type == SPK_VALUES_F32) {
      if (uotk) launch_tiled<true, true, float>(ctx, A);
      else launch_tiled<true, false, float>(ctx, A);
    } else {
      if (uotk) launch_tiled<true, true, double>(ctx, A);
      else launch_tiled<true, false, double>(ctx, A);
    }
    unsigned int overflow = 0;
    download(ctx, &overflow, ovf, sizeof overflow);
    if (!overflow) {
      int_to_ll_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(rcnt.as<int>(), n, capll.as<long long>());
      ++ctx->launches;
      SPK_CUDA(cudaMemsetAsync(sk->row_ptr.p, 0, sizeof(long long), ctx->stream));
      SPK_CUDA(cub::DeviceScan::InclusiveSum(ctx->scratch.p, tb, capll.as<long long>(), sk->row_ptr.as<long long>() + 1,
                                             (int)n, ctx->stream));
      long long nnz = 0;
      SPK_CUDA(cudaMemcpyAsync(&nnz, sk->row_ptr.as<long long>() + n, sizeof nnz, cudaMemcpyDeviceToHost,
                               ctx->stream));
      SPK_CUDA(cudaStreamSynchronize(ctx->stream));
      if (nnz > 0xffffffffLL) fail(SPK_E_BUDGET_TOO_LARGE, "sketch exceeds 2^32 entries");
      sk->nnz = nnz;
      sk->col_idx.alloc(sizeof(uint32_t) * std::max<long long>(nnz, 1));
      sk->values.alloc(vbytes * std::max<long long>(nnz, 1));
      static const bool dbg = std::getenv("SPK_DEBUG_TIMING") != nullptr;
      std::unique_ptr<Timer> tq(dbg ? new Timer(ctx->stream) : nullptr);
      compact_kernel<<<grid_for_rows(ctx, n, 8), 256, 0, ctx->stream>>>(
          n, off.as<long long>(), sk->row_ptr.as<long long>(), pcol.as<uint32_t>(), pval.as<unsigned char>(),
          (int)vbytes, sk->col_idx.as<uint32_t>(), sk->values.as<unsigned char>());
      ++ctx->launches;
      SPK_CUDA(cudaGetLastError());
      if (tq) {
        std::fprintf(stderr, "[timing]   compact %.4f s\n", tq->stop());
        tq.reset(new Timer(ctx->stream));
      }
      build_csc(ctx, sk);
      if (tq) {
        std::fprintf(stderr, "[timing]   build_csc %.4f s\n", tq->stop());
        tq.reset(new Timer(ctx->stream));
      }
      sk->kernel_mean = sketch_kernel_mean(ctx, sk);
      if (tq) std::fprintf(stderr, "[timing]   kernel_mean %.4f s\n", tq->stop());
      return;
    }
    // a row outgrew its slot: redo exactly with the two-pass kernels below
  }

  DBuf cnt(sizeof(long long) * n);
  const int grid = grid_for_rows(ctx, n, 8);
  sample_rows_kernel<false, double><<<grid, 256, 0, ctx->stream>>>(S, P, s, seed, row0, n, cnt.as<long long>(),
                                                                   nullptr, nullptr, nullptr);
  ++ctx->launches;
  // row_ptr = exclusive scan of counts, row_ptr[n] = nnz
  SPK_CUDA(cudaMemsetAsync(sk->row_ptr.p, 0, sizeof(long long), ctx->stream));
  size_t tmp_bytes = 0;
  SPK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, cnt.as<long long>(), sk->row_ptr.as<long long>() + 1,
                                         (int)n, ctx->stream));
  ctx->scratch.ensure(tmp_bytes);
  SPK_CUDA(cub::DeviceScan::InclusiveSum(ctx->scratch.p, tmp_bytes, cnt.as<long long>(),
                                         sk->row_ptr.as<long long>() + 1, (int)n, ctx->stream));
  ++ctx->launches;
  long long nnz = 0;
  SPK_CUDA(cudaMemcpyAsync(&nnz, sk->row_ptr.as<long long>() + n, sizeof nnz, cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (nnz > 0xffffffffLL) fail(SPK_E_BUDGET_TOO_LARGE, "sketch exceeds 2^32 entries");
  sk->nnz = nnz;
  sk->col_idx.alloc(sizeof(uint32_t) * std::max<long long>(nnz, 1));
  sk->values.alloc(vbytes * std::max<long long>(nnz, 1));
  if (value_type == SPK_VALUES_F32)
    sample_rows_kernel<true, float><<<grid, 256, 0, ctx->stream>>>(S, P, s, seed, row0, n, nullptr,
                                                                   sk->row_ptr.as<long long>(),
                                                                   sk->col_idx.as<uint32_t>(), sk->values.as<float>());
  else
    sample_rows_kernel<true, double><<<grid, 256, 0, ctx->stream>>>(S, P, s, seed, row0, n, nullptr,
                                                                    sk->row_ptr.as<long long>(),
                                                                    sk->col_idx.as<uint32_t>(),
                                                                    sk->values.as<double>());
  ++ctx->launches;
  SPK_CUDA(cudaGetLastError());
  build_csc(ctx, sk);
  sk->kernel_mean = sketch_kernel_mean(ctx, sk);
}

void build_csc(spk_ctx* ctx, spk_sketch* sk) {
  const int64_t n = sk->n, m = sk->nnz;
  const int64_t nc = sk->n_cols ? sk->n_cols : n;  // columns
  const size_t vbytes = sk->value_type == SPK_VALUES_F32 ? 4 : 8;
  sk->col_ptr.alloc(sizeof(long long) * (nc + 1));
  sk->row_idx.alloc(sizeof(uint32_t) * std::max<int64_t>(m, 1));
  sk->values_t.alloc(vbytes * std::max<int64_t>(m, 1));
  DBuf cnt(sizeof(long long) * nc);
  SPK_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes, ctx->stream));
  SPK_CUDA(cudaMemsetAsync(sk->col_ptr.p, 0, sizeof(long long), ctx->stream));
  if (m > 0) {
    DBuf &iota = tmp_buf(ctx, 0, sizeof(uint32_t) * m), &perm = tmp_buf(ctx, 1, sizeof(uint32_t) * m),
         &rows = tmp_buf(ctx, 2, sizeof(uint32_t) * m), &keys_out = tmp_buf(ctx, 3, sizeof(uint32_t) * m);
    expand_rows_kernel<<<grid_for_rows(ctx, n, 8), 256, 0, ctx->stream>>>(sk->row_ptr.as<long long>(), n,
                                                                           rows.as<uint32_t>());
    iota_kernel<<<grid_for(ctx, m, 256), 256, 0, ctx->stream>>>(iota.as<uint32_t>(), m);
    col_count_kernel<<<grid_for(ctx, m, 256), 256, 0, ctx->stream>>>(sk->col_idx.as<uint32_t>(), m,
                                                                     cnt.as<long long>());
    ctx->launches += 3;
    int end_bit = 1;
    while ((int64_t(1) << end_bit) < nc) ++end_bit;
    size_t tmp_bytes = 0;
    // Stable LSD radix sort by column: equal columns keep CSR (row-major)
    // order, i.e. rows ascend inside each column as spmv_t visits them.
    SPK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, sk->col_idx.as<uint32_t>(),
                                             keys_out.as<uint32_t>(), iota.as<uint32_t>(), perm.as<uint32_t>(),
                                             (int)m, 0, end_bit, ctx->stream));
    ctx->scratch.ensure(tmp_bytes);
    SPK_CUDA(cub::DeviceRadixSort::SortPairs(ctx->scratch.p, tmp_bytes, sk->col_idx.as<uint32_t>(),
                                             keys_out.as<uint32_t>(), iota.as<uint32_t>(), perm.as<uint32_t>(),
                                             (int)m, 0, end_bit, ctx->stream));
    ++ctx->launches;
    if (sk->value_type == SPK_VALUES_F32)
      gather_csc_kernel<float><<<grid_for(ctx, m, 256), 256, 0, ctx->stream>>>(
          perm.as<uint32_t>(), rows.as<uint32_t>(), sk->values.as<float>(), m, sk->row_idx.as<uint32_t>(),
          sk->values_t.as<float>());
    else
      gather_csc_kernel<double><<<grid_for(ctx, m, 256), 256, 0, ctx->stream>>>(
          perm.as<uint32_t>(), rows.as<uint32_t>(), sk->values.as<double>(), m, sk->row_idx.as<uint32_t>(),
          sk->values_t.as<double>());
    ++ctx->launches;
  }
  size_t tmp_bytes = 0;
  SPK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, cnt.as<long long>(), sk->col_ptr.as<long long>() + 1,
                                         (int)nc, ctx->stream));
  ctx->scratch.ensure(tmp_bytes);
  SPK_CUDA(cub::DeviceScan::InclusiveSum(ctx->scratch.p, tmp_bytes, cnt.as<long long>(),
                                         sk->col_ptr.as<long long>() + 1, (int)nc, ctx->stream));
  ++ctx->launches;
  SPK_CUDA(cudaGetLastError());
}

// kernel_mean (solvers.cpp:172-177): sum of sketch values / n^2.
double sketch_kernel_mean(spk_ctx* ctx, spk_sketch* sk) {
  const int64_t m = sk->nnz;
  double acc = 0.0;
  if (m > 0) {
    if (ctx->deterministic) {
      DBuf out(sizeof(double));
      if (sk->value_type == SPK_VALUES_F32)
        sum_values_seq_kernel<float><<<1, 1, 0, ctx->stream>>>(sk->values.as<float>(), m, out.as<double>());
      else
        sum_values_seq_kernel<double><<<1, 1, 0, ctx->stream>>>(sk->values.as<double>(), m, out.as<double>());
      ++ctx->launches;
      download(ctx, &acc, out, sizeof acc);
    } else {
      const int grid = grid_for(ctx, m, 256);
      DBuf part(sizeof(double) * grid), out(sizeof(double));
      if (sk->value_type == SPK_VALUES_F32)
        sum_values_kernel<float><<<grid, 256, 0, ctx->stream>>>(sk->values.as<float>(), m, part.as<double>());
      else
        sum_values_kernel<double><<<grid, 256, 0, ctx->stream>>>(sk->values.as<double>(), m, part.as<double>());
      reduce_rows_kernel<double><<<1, 1024, 0, ctx->stream>>>(part.as<double>(), grid, out.as<double>());
      ctx->launches += 2;
      download(ctx, &acc, out, sizeof acc);
    }
  }
  // A row shard holds a partial sum of the full n x n estimate; shards add up.
  const double nd = static_cast<double>(sk->n_cols ? sk->n_cols : sk->n);
  return acc / (nd * nd);
}

}  // namespace spk
