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
#include <cmath>
#include <cstring>

#include "common.cuh"
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
  return isinf(c) ? 0.0 : exp(-c / S.eps);
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
__global__ void sample_rows_kernel(KSrc S, DPlan P, double s, uint64_t seed, long long* row_cnt,
                                   const long long* row_ptr, uint32_t* col_out, VT* val_out) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < S.n; i += nwarps) {
    const uint64_t state0 = mix_seed(seed, (uint64_t)i);
    uint64_t base_t = 0;
    long long cnt = 0;
    const long long out0 = EMIT ? row_ptr[i] : 0;
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
    if (!EMIT && lane == 0) row_cnt[i] = cnt;
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
    kern[q] = isinf(c) ? 0.0 : exp(-c / S.eps);
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

}  // namespace

// ---- host orchestration ----------------------------------------------------------

void make_dev_kernel(spk_ctx* ctx, const spk_kernel_desc* kd, double default_eps, DevKernel& dk,
                     bool need_cost) {
  if (!kd) fail(SPK_E_LENGTH_MISMATCH, "null kernel descriptor");
  const int64_t n = kd->n;
  if (n <= 0) fail(SPK_E_LENGTH_MISMATCH, "kernel dimension must be positive");
  dk.n = n;
  dk.eps = kd->kernel_epsilon > 0.0 ? kd->kernel_epsilon : default_eps;
  if (kd->K) {
    dk.dense = true;
    dk.nnz_ratio = kd->nnz_ratio;
    upload(ctx, dk.K, kd->K, sizeof(double) * n * n);
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
  dk.have_cost = true;
  if (kd->cost_scale > 0.0) {
    dk.scale = kd->cost_scale;
  } else {
    // c0 = max finite cost (geometry.cpp:61), the configs' max-normalisation.
    DBuf m(sizeof(unsigned long long));
    SPK_CUDA(cudaMemsetAsync(m.p, 0, m.bytes, ctx->stream));
    dk.scale = 1.0;
    KSrc S = make_src(dk);
    max_cost_kernel<<<grid_for(ctx, n * n, 256), 256, 0, ctx->stream>>>(S, m.as<unsigned long long>());
    ++ctx->launches;
    unsigned long long bits = 0;
    SPK_CUDA(cudaMemcpyAsync(&bits, m.p, sizeof bits, cudaMemcpyDeviceToHost, ctx->stream));
    SPK_CUDA(cudaStreamSynchronize(ctx->stream));
    double c0;
    std::memcpy(&c0, &bits, sizeof c0);
    dk.scale = c0;
    dk.max_normalised = true;
  }
}

void build_plan(spk_ctx* ctx, DevKernel& dk, const double* a, const double* b, int plan_kind,
                double lambda, double eps, double theta, PlanInfo& plan) {
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
    for (int64_t i = 0; i < n; ++i) plan.row_w[i] = std::pow(a[i], g_ab);
    for (int64_t j = 0; j < n; ++j) plan.col_w[j] = std::pow(b[j], g_ab);
  } else if (plan_kind == SPK_PLAN_BARYCENTER) {  // sparsify.cpp:122-128
    double sb = 0.0;
    for (int64_t j = 0; j < n; ++j) sb += (plan.col_w[j] = std::sqrt(b[j]));
    zero_mass = (sb == 0.0);
    for (int64_t j = 0; j < n; ++j) plan.col_w[j] /= sb;
    for (int64_t i = 0; i < n; ++i) plan.row_w[i] = 1.0 / static_cast<double>(n);
  } else {  // uniform, sparsify.cpp:144
    for (int64_t i = 0; i < n; ++i) plan.row_w[i] = plan.col_w[i] = 1.0 / static_cast<double>(n);
  }

  // ---- support size and grid normaliser (device pass over n^2 entries) ----
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
  long long support = static_cast<long long>(n) * n;
  double total = 0.0;
  if (need_pass) {
    DBuf rw, cw;
    upload(ctx, rw, plan.row_w.data(), sizeof(double) * n);
    upload(ctx, cw, plan.col_w.data(), sizeof(double) * n);
    DPlan P{};
    P.row_w = rw.as<double>();
    P.col_w = cw.as<double>();
    P.kind = plan_kind;
    P.g_k = plan.g_k;
    DBuf rn(sizeof(long long) * n), rs(sizeof(double) * n), tot(sizeof(double)), tn(sizeof(long long));
    KSrc S = make_src(dk);
    plan_rows_kernel<<<grid_for_rows(ctx, n, 8), 256, 0, ctx->stream>>>(S, P, rn.as<long long>(),
                                                                         rs.as<double>());
    reduce_rows_kernel<double><<<1, 1024, 0, ctx->stream>>>(rs.as<double>(), n, tot.as<double>());
    reduce_rows_kernel<long long><<<1, 1024, 0, ctx->stream>>>(rn.as<long long>(), n, tn.as<long long>());
    ctx->launches += 3;
    SPK_CUDA(cudaMemcpyAsync(&total, tot.p, sizeof total, cudaMemcpyDeviceToHost, ctx->stream));
    SPK_CUDA(cudaMemcpyAsync(&support, tn.p, sizeof support, cudaMemcpyDeviceToHost, ctx->stream));
    SPK_CUDA(cudaStreamSynchronize(ctx->stream));
  }
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
                   int value_type, spk_sketch* sk) {
  const int64_t n = dk.n;
  const double nn = static_cast<double>(n) * static_cast<double>(n);
  if (!(s > 0.0) || s >= nn) fail(SPK_E_BUDGET_TOO_LARGE, "budget s must satisfy 0 < s < n^2");
  DBuf rw, cw;
  upload(ctx, rw, plan.row_w.data(), sizeof(double) * n);
  upload(ctx, cw, plan.col_w.data(), sizeof(double) * n);
  DPlan P = device_plan(plan, rw.as<double>(), cw.as<double>());
  KSrc S = make_src(dk);

  sk->n = n;
  sk->seed = seed;
  sk->value_type = value_type;
  sk->kernel_nnz = plan.kernel_nnz;
  sk->factorized_plan = plan.factorized ? 1 : 0;
  sk->row_ptr.alloc(sizeof(long long) * (n + 1));
  DBuf cnt(sizeof(long long) * n);
  const int grid = grid_for_rows(ctx, n, 8);
  sample_rows_kernel<false, double><<<grid, 256, 0, ctx->stream>>>(S, P, s, seed, cnt.as<long long>(),
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
  const size_t vbytes = value_type == SPK_VALUES_F32 ? 4 : 8;
  sk->col_idx.alloc(sizeof(uint32_t) * std::max<long long>(nnz, 1));
  sk->values.alloc(vbytes * std::max<long long>(nnz, 1));
  if (value_type == SPK_VALUES_F32)
    sample_rows_kernel<true, float><<<grid, 256, 0, ctx->stream>>>(
        S, P, s, seed, nullptr, sk->row_ptr.as<long long>(), sk->col_idx.as<uint32_t>(), sk->values.as<float>());
  else
    sample_rows_kernel<true, double><<<grid, 256, 0, ctx->stream>>>(
        S, P, s, seed, nullptr, sk->row_ptr.as<long long>(), sk->col_idx.as<uint32_t>(), sk->values.as<double>());
  ++ctx->launches;
  SPK_CUDA(cudaGetLastError());
  build_csc(ctx, sk);
  sk->kernel_mean = sketch_kernel_mean(ctx, sk);
}

void build_csc(spk_ctx* ctx, spk_sketch* sk) {
  const int64_t n = sk->n, m = sk->nnz;
  const size_t vbytes = sk->value_type == SPK_VALUES_F32 ? 4 : 8;
  sk->col_ptr.alloc(sizeof(long long) * (n + 1));
  sk->row_idx.alloc(sizeof(uint32_t) * std::max<int64_t>(m, 1));
  sk->values_t.alloc(vbytes * std::max<int64_t>(m, 1));
  DBuf cnt(sizeof(long long) * n);
  SPK_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes, ctx->stream));
  SPK_CUDA(cudaMemsetAsync(sk->col_ptr.p, 0, sizeof(long long), ctx->stream));
  if (m > 0) {
    DBuf rows(sizeof(uint32_t) * m), keys_out(sizeof(uint32_t) * m), iota(sizeof(uint32_t) * m),
        perm(sizeof(uint32_t) * m);
    expand_rows_kernel<<<grid_for_rows(ctx, n, 8), 256, 0, ctx->stream>>>(sk->row_ptr.as<long long>(), n,
                                                                           rows.as<uint32_t>());
    iota_kernel<<<grid_for(ctx, m, 256), 256, 0, ctx->stream>>>(iota.as<uint32_t>(), m);
    col_count_kernel<<<grid_for(ctx, m, 256), 256, 0, ctx->stream>>>(sk->col_idx.as<uint32_t>(), m,
                                                                     cnt.as<long long>());
    ctx->launches += 3;
    int end_bit = 1;
    while ((int64_t(1) << end_bit) < n) ++end_bit;
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
                                         (int)n, ctx->stream));
  ctx->scratch.ensure(tmp_bytes);
  SPK_CUDA(cub::DeviceScan::InclusiveSum(ctx->scratch.p, tmp_bytes, cnt.as<long long>(),
                                         sk->col_ptr.as<long long>() + 1, (int)n, ctx->stream));
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
  const double nd = static_cast<double>(sk->n);
  return acc / (nd * nd);
}

}  // namespace spk
