// readout.cu -- fused plan readout (north-star item 4).
//
// Reference semantics: TransportPlan::for_each_entry (include/sparsink/solvers.hpp:234-252)
// visits (i, j, T_ij) with T_ij = u_i K~_ij v_j (log: exp(lu + log K~ + lv)) only where
// T_ij > 0; row_marginal / col_marginal (proj/src/solvers.cpp:215-225);
// transport_and_entropy (:265-276) with InfiniteCostOnSupport; ot_objective /
// uot_objective (:280-293); kl_divergence (:246-260); residuals
// (solvers.hpp:380-389). One pass over the CSR gives row marginals, <T, C>
// and H(T) per row (costs recomputed from coordinates, no n^2 storage); one
// pass over the CSC gives column marginals in the reference's summation
// order. Deterministic mode sums sequentially in the reference's order.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "internal.h"
#include "ksrc.cuh"

namespace spk {

namespace {

template <bool LOG>
__device__ __forceinline__ double plan_entry(double ui, double k, double vj) {
  if (LOG) {
    if (ui == -CUDART_INF || vj == -CUDART_INF) return 0.0;
    return exp(dadd(dadd(ui, log(k)), vj));
  }
  return dmul(dmul(ui, k), vj);
}

// Row pass: row marginal, <T,C> and entropy per row (warp per row).
template <bool LOG, bool OBJ, class VT>
__global__ void row_pass_kernel(int64_t n, const long long* ptr, const uint32_t* idx, const VT* val,
                                const double* u, const double* v, CostSrc cs, double* row_m, double* row_c,
                                double* row_h, unsigned long long* inf_flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    double m = 0.0, c = 0.0, h = 0.0;
    const double ui = u[i];
    for (long long p = ptr[i] + lane; p < ptr[i + 1]; p += 32) {
      const int64_t j = idx[p];
      const double t = plan_entry<LOG>(ui, (double)val[p], v[j]);
      if (!(t > 0.0)) continue;
      m += t;
      if (OBJ) {
        const double cij = cs(i, j);
        if (isinf(cij)) atomicMin(inf_flag, (unsigned long long)i);
        c = dadd(c, dmul(t, cij));
        h = dsub(h, dmul(t, dsub(log(t), 1.0)));
      }
    }
    m = warp_sum(m);
    if (OBJ) {
      c = warp_sum(c);
      h = warp_sum(h);
    }
    if (lane == 0) {
      row_m[i] = m;
      if (OBJ) {
        row_c[i] = c;
        row_h[i] = h;
      }
    }
  }
}

// Column pass over the CSC (rows ascending) -> column marginals.
template <bool LOG, bool DET, class VT>
__global__ void col_pass_kernel(int64_t n, const long long* ptr, const uint32_t* idx, const VT* val,
                                const double* u, const double* v, double* col_m) {
  if (DET) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
      double m = 0.0;
      const double vj = v[j];
      for (long long p = ptr[j]; p < ptr[j + 1]; ++p) {
        const double t = plan_entry<LOG>(u[idx[p]], (double)val[p], vj);
        if (t > 0.0) m = dadd(m, t);
      }
      col_m[j] = m;
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nw) {
    double m = 0.0;
    const double vj = v[j];
    for (long long p = ptr[j] + lane; p < ptr[j + 1]; p += 32) {
      const double t = plan_entry<LOG>(u[idx[p]], (double)val[p], vj);
      if (t > 0.0) m += t;
    }
    m = warp_sum(m);
    if (lane == 0) col_m[j] = m;
  }
}

// Deterministic: row marginals per row and <T,C>, H(T) as ONE running sum in
// row-major order (transport_and_entropy visits entries sequentially).
template <bool LOG, bool OBJ, class VT>
__global__ void row_seq_kernel(int64_t n, const long long* ptr, const uint32_t* idx, const VT* val,
                               const double* u, const double* v, CostSrc cs, double* row_m, double* sums,
                               unsigned long long* inf_flag) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double c = 0.0, h = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double m = 0.0;
    for (long long p = ptr[i]; p < ptr[i + 1]; ++p) {
      const int64_t j = idx[p];
      const double t = plan_entry<LOG>(u[i], (double)val[p], v[j]);
      if (!(t > 0.0)) continue;
      m = dadd(m, t);
      if (OBJ) {
        const double cij = cs(i, j);
        if (isinf(cij)) {
          atomicMin(inf_flag, (unsigned long long)i);
          continue;
        }
        c = dadd(c, dmul(t, cij));
        h = dsub(h, dmul(t, dsub(log(t), 1.0)));
      }
    }
    row_m[i] = m;
  }
  sums[0] = c;
  sums[1] = h;
}

// Elementwise terms: |m - w| (mode 0) or the KL term (mode 1, solvers.cpp:250-257).
__global__ void terms_kernel(int64_t n, const double* m, const double* w, int mode, double* out,
                             unsigned long long* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = m[i], y = w[i];
    if (mode == 0) {
      out[i] = fabs(dsub(x, y));
    } else if (x > 0.0) {
      if (y <= 0.0) atomicMin(bad, (unsigned long long)i);
      out[i] = dadd(dsub(dmul(x, log(x / y)), x), y);
    } else {
      out[i] = y;
    }
  }
}

__global__ void seq_sum_kernel(const double* v, int64_t n, double* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double acc = 0.0;
  for (int64_t k = 0; k < n; ++k) acc = dadd(acc, v[k]);
  *out = acc;
}

__global__ void tree_sum_kernel(const double* v, int64_t n, double* out) {
  __shared__ double sm[1024];
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * per;
  const int64_t e = b + per < n ? b + per : n;
  double acc = 0.0;
  for (int64_t k = b; k < e; ++k) acc += v[k];
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

__global__ void fill_u64(unsigned long long* p, unsigned long long v) { *p = v; }

int rows_grid(spk_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, (int64_t)ctx->num_sms * 16));
}
int elem_grid(spk_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8));
}

double sum_array(spk_ctx* ctx, const double* v, int64_t n, DBuf& tmp) {
  tmp.ensure(sizeof(double));
  if (ctx->deterministic) seq_sum_kernel<<<1, 1, 0, ctx->stream>>>(v, n, tmp.as<double>());
  else tree_sum_kernel<<<1, 1024, 0, ctx->stream>>>(v, n, tmp.as<double>());
  ++ctx->launches;
  double r = 0.0;
  download(ctx, &r, tmp, sizeof r);
  return r;
}

// Marginal residuals + KL + objective assembly from device marginals.
void finish(spk_ctx* ctx, ReadWs& R, int64_t n, const double* row_m, const double* col_m, const double* a,
            const double* b, bool want_obj, int uot, double lambda, double eps, double cost, double entropy,
            ReadoutOut& out) {
  R.terms.ensure(sizeof(double) * n);
  R.bad.ensure(sizeof(unsigned long long));
  DBuf& terms = R.terms;
  DBuf& tmp = R.tmp;
  DBuf& bad = R.bad;
  const int g = elem_grid(ctx, n);
  terms_kernel<<<g, 256, 0, ctx->stream>>>(n, row_m, a, 0, terms.as<double>(), nullptr);
  ++ctx->launches;
  out.residual_row = sum_array(ctx, terms.as<double>(), n, tmp);
  terms_kernel<<<g, 256, 0, ctx->stream>>>(n, col_m, b, 0, terms.as<double>(), nullptr);
  ++ctx->launches;
  out.residual_col = sum_array(ctx, terms.as<double>(), n, tmp);
  if (!want_obj) return;
  if (!uot) {
    out.objective = cost - eps * entropy;  // ot_objective (solvers.cpp:280-284)
  } else {
    fill_u64<<<1, 1, 0, ctx->stream>>>(bad.as<unsigned long long>(), ~0ull);
    terms_kernel<<<g, 256, 0, ctx->stream>>>(n, row_m, a, 1, terms.as<double>(), bad.as<unsigned long long>());
    ctx->launches += 2;
    const double kl_a = sum_array(ctx, terms.as<double>(), n, tmp);
    unsigned long long flag = 0;
    download(ctx, &flag, bad, sizeof flag);
    if (flag != ~0ull) fail(SPK_E_ERROR, "KL undefined: mass off support");
    terms_kernel<<<g, 256, 0, ctx->stream>>>(n, col_m, b, 1, terms.as<double>(), bad.as<unsigned long long>());
    ++ctx->launches;
    const double kl_b = sum_array(ctx, terms.as<double>(), n, tmp);
    download(ctx, &flag, bad, sizeof flag);
    if (flag != ~0ull) fail(SPK_E_ERROR, "KL undefined: mass off support");
    // uot_objective (solvers.cpp:286-293), evaluated left to right
    out.objective = cost + lambda * kl_a + lambda * kl_b - eps * entropy;
  }
  out.have_objective = true;
}

template <bool LOG, class VT>
void sparse_readout_t(spk_ctx* ctx, spk_sketch* sk, DevKernel* dk, const double* u, const double* v,
                      const double* a, const double* b, bool want_obj, int uot, double lambda, double eps,
                      double* row_m_host, double* col_m_host, ReadoutOut& out) {
  const int64_t n = sk->n;
  cudaStream_t s = ctx->stream;
  ReadWs& R = sk->rws;
  R.row_m.ensure(sizeof(double) * n);
  R.col_m.ensure(sizeof(double) * n);
  R.flag.ensure(sizeof(unsigned long long));
  R.sums.ensure(2 * sizeof(double));
  DBuf& row_m = R.row_m;
  DBuf& col_m = R.col_m;
  DBuf& flag = R.flag;
  DBuf& tmp = R.tmp;
  fill_u64<<<1, 1, 0, s>>>(flag.as<unsigned long long>(), ~0ull);
  ++ctx->launches;
  const CostSrc cs = cost_src_of(dk);
  const bool obj = want_obj && dk && dk->have_cost;
  double cost = 0.0, entropy = 0.0;
  if (ctx->deterministic) {
    DBuf& sums = R.sums;
    if (obj)
      row_seq_kernel<LOG, true, VT><<<1, 1, 0, s>>>(n, sk->row_ptr.as<long long>(), sk->col_idx.as<uint32_t>(),
                                                     sk->values.as<VT>(), u, v, cs, row_m.as<double>(),
                                                     sums.as<double>(), flag.as<unsigned long long>());
    else
      row_seq_kernel<LOG, false, VT><<<1, 1, 0, s>>>(n, sk->row_ptr.as<long long>(), sk->col_idx.as<uint32_t>(),
                                                      sk->values.as<VT>(), u, v, cs, row_m.as<double>(),
                                                      sums.as<double>(), flag.as<unsigned long long>());
    col_pass_kernel<LOG, true, VT><<<elem_grid(ctx, n), 256, 0, s>>>(
        n, sk->col_ptr.as<long long>(), sk->row_idx.as<uint32_t>(), sk->values_t.as<VT>(), u, v, col_m.as<double>());
    ctx->launches += 2;
    double hs[2];
    download(ctx, hs, sums, sizeof hs);
    cost = hs[0];
    entropy = hs[1];
  } else {
    R.row_c.ensure(sizeof(double) * n);
    R.row_h.ensure(sizeof(double) * n);
    DBuf& row_c = R.row_c;
    DBuf& row_h = R.row_h;
    if (obj)
      row_pass_kernel<LOG, true, VT><<<rows_grid(ctx, n), 256, 0, s>>>(
          n, sk->row_ptr.as<long long>(), sk->col_idx.as<uint32_t>(), sk->values.as<VT>(), u, v, cs,
          row_m.as<double>(), row_c.as<double>(), row_h.as<double>(), flag.as<unsigned long long>());
    else
      row_pass_kernel<LOG, false, VT><<<rows_grid(ctx, n), 256, 0, s>>>(
          n, sk->row_ptr.as<long long>(), sk->col_idx.as<uint32_t>(), sk->values.as<VT>(), u, v, cs,
          row_m.as<double>(), row_c.as<double>(), row_h.as<double>(), flag.as<unsigned long long>());
    col_pass_kernel<LOG, false, VT><<<rows_grid(ctx, n), 256, 0, s>>>(
        n, sk->col_ptr.as<long long>(), sk->row_idx.as<uint32_t>(), sk->values_t.as<VT>(), u, v, col_m.as<double>());
    ctx->launches += 2;
    if (obj) {
      cost = sum_array(ctx, row_c.as<double>(), n, tmp);
      entropy = sum_array(ctx, row_h.as<double>(), n, tmp);
    }
  }
  if (obj) {
    unsigned long long f = 0;
    download(ctx, &f, flag, sizeof f);
    if (f != ~0ull) fail(SPK_E_INFINITE_COST_ON_SUPPORT, "plan mass on a blocked entry");
  }
  finish(ctx, R, n, row_m.as<double>(), col_m.as<double>(), a, b, obj, uot, lambda, eps, cost, entropy, out);
  if (row_m_host) download(ctx, row_m_host, row_m, sizeof(double) * n);
  if (col_m_host) download(ctx, col_m_host, col_m, sizeof(double) * n);
}

}  // namespace

void sparse_readout(spk_ctx* ctx, spk_sketch* sk, DevKernel* dk, int log_domain, const double* a, const double* b,
                    bool want_objective, int uot, double lambda, double eps, double* row_m_host,
                    double* col_m_host, ReadoutOut& out) {
  const double* u = log_domain ? sk->lu.as<double>() : sk->u.as<double>();
  const double* v = log_domain ? sk->lv.as<double>() : sk->v.as<double>();
  if (sk->value_type == SPK_VALUES_F32) {
    if (log_domain)
      sparse_readout_t<true, float>(ctx, sk, dk, u, v, a, b, want_objective, uot, lambda, eps, row_m_host, col_m_host, out);
    else
      sparse_readout_t<false, float>(ctx, sk, dk, u, v, a, b, want_objective, uot, lambda, eps, row_m_host, col_m_host, out);
  } else {
    if (log_domain)
      sparse_readout_t<true, double>(ctx, sk, dk, u, v, a, b, want_objective, uot, lambda, eps, row_m_host, col_m_host, out);
    else
      sparse_readout_t<false, double>(ctx, sk, dk, u, v, a, b, want_objective, uot, lambda, eps, row_m_host, col_m_host, out);
  }
}


// ---- dense readout (KernelMatrix or K recomputed from coordinates) ----------

namespace {

template <bool LOG, bool OBJ, class KF>
__global__ void dense_row_pass_kernel(KF k, int64_t n, const double* u, const double* v, CostSrc cs, double* row_m,
                                      double* row_c, double* row_h, unsigned long long* inf_flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    double m = 0.0, c = 0.0, h = 0.0;
    const double ui = u[i];
    for (int64_t j = lane; j < n; j += 32) {
      const double kij = k(i, j);
      if (!(kij > 0.0)) continue;  // kernel_for_each visits K > 0 only (solvers.hpp:116-123)
      const double t = plan_entry<LOG>(ui, kij, v[j]);
      if (!(t > 0.0)) continue;
      m += t;
      if (OBJ) {
        const double cij = cs(i, j);
        if (isinf(cij)) atomicMin(inf_flag, (unsigned long long)i);
        c = dadd(c, dmul(t, cij));
        h = dsub(h, dmul(t, dsub(log(t), 1.0)));
      }
    }
    m = warp_sum(m);
    if (OBJ) {
      c = warp_sum(c);
      h = warp_sum(h);
    }
    if (lane == 0) {
      row_m[i] = m;
      if (OBJ) {
        row_c[i] = c;
        row_h[i] = h;
      }
    }
  }
}

template <bool LOG, class KF>
__global__ void dense_col_pass_kernel(KF k, int64_t n, const double* u, const double* v, double* col_m) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double m = 0.0;
    const double vj = v[j];
    for (int64_t i = 0; i < n; ++i) {
      const double kij = k(i, j);
      if (!(kij > 0.0)) continue;
      const double t = plan_entry<LOG>(u[i], kij, vj);
      if (t > 0.0) m = dadd(m, t);
    }
    col_m[j] = m;
  }
}

template <bool LOG, bool OBJ, class KF>
__global__ void dense_row_seq_kernel(KF k, int64_t n, const double* u, const double* v, CostSrc cs, double* row_m,
                                     double* sums, unsigned long long* inf_flag) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double c = 0.0, h = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double m = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      const double kij = k(i, j);
      if (!(kij > 0.0)) continue;
      const double t = plan_entry<LOG>(u[i], kij, v[j]);
      if (!(t > 0.0)) continue;
      m = dadd(m, t);
      if (OBJ) {
        const double cij = cs(i, j);
        if (isinf(cij)) {
          atomicMin(inf_flag, (unsigned long long)i);
          continue;
        }
        c = dadd(c, dmul(t, cij));
        h = dsub(h, dmul(t, dsub(log(t), 1.0)));
      }
    }
    row_m[i] = m;
  }
  sums[0] = c;
  sums[1] = h;
}

template <bool LOG, class KF>
void dense_readout_t(spk_ctx* ctx, KF kf, DevKernel& dk, const double* u, const double* v, const double* a,
                     const double* b, bool want_obj, int uot, double lambda, double eps, ReadoutOut& out,
                     double* row_m_host, double* col_m_host) {
  const int64_t n = dk.n;
  cudaStream_t s = ctx->stream;
  DBuf row_m(sizeof(double) * n), col_m(sizeof(double) * n), flag(sizeof(unsigned long long)), tmp;
  fill_u64<<<1, 1, 0, s>>>(flag.as<unsigned long long>(), ~0ull);
  ++ctx->launches;
  const CostSrc cs = cost_src_of(&dk);
  const bool obj = want_obj && dk.have_cost;
  double cost = 0.0, entropy = 0.0;
  if (ctx->deterministic) {
    DBuf sums(2 * sizeof(double));
    if (obj)
      dense_row_seq_kernel<LOG, true, KF><<<1, 1, 0, s>>>(kf, n, u, v, cs, row_m.as<double>(), sums.as<double>(),
                                                          flag.as<unsigned long long>());
    else
      dense_row_seq_kernel<LOG, false, KF><<<1, 1, 0, s>>>(kf, n, u, v, cs, row_m.as<double>(), sums.as<double>(),
                                                           flag.as<unsigned long long>());
    ++ctx->launches;
    double hs[2];
    download(ctx, hs, sums, sizeof hs);
    cost = hs[0];
    entropy = hs[1];
  } else {
    DBuf row_c(sizeof(double) * n), row_h(sizeof(double) * n);
    if (obj)
      dense_row_pass_kernel<LOG, true, KF><<<rows_grid(ctx, n), 256, 0, s>>>(
          kf, n, u, v, cs, row_m.as<double>(), row_c.as<double>(), row_h.as<double>(), flag.as<unsigned long long>());
    else
      dense_row_pass_kernel<LOG, false, KF><<<rows_grid(ctx, n), 256, 0, s>>>(
          kf, n, u, v, cs, row_m.as<double>(), row_c.as<double>(), row_h.as<double>(), flag.as<unsigned long long>());
    ++ctx->launches;
    if (obj) {
      cost = sum_array(ctx, row_c.as<double>(), n, tmp);
      entropy = sum_array(ctx, row_h.as<double>(), n, tmp);
    }
  }
  dense_col_pass_kernel<LOG, KF><<<elem_grid(ctx, n), 256, 0, s>>>(kf, n, u, v, col_m.as<double>());
  ++ctx->launches;
  if (obj) {
    unsigned long long f = 0;
    download(ctx, &f, flag, sizeof f);
    if (f != ~0ull) fail(SPK_E_INFINITE_COST_ON_SUPPORT, "plan mass on a blocked entry");
  }
  ReadWs R;
  finish(ctx, R, n, row_m.as<double>(), col_m.as<double>(), a, b, obj, uot, lambda, eps, cost, entropy, out);
  if (row_m_host) download(ctx, row_m_host, row_m, sizeof(double) * n);
  if (col_m_host) download(ctx, col_m_host, col_m, sizeof(double) * n);
}

}  // namespace

void dense_readout(spk_ctx* ctx, DevKernel& dk, int log_domain, const DBuf& u, const DBuf& v, const DBuf& lu,
                   const DBuf& lv, const double* a, const double* b, bool want_objective, int uot, double lambda,
                   double eps, ReadoutOut& out, double* rmh, double* cmh) {
  const double* pu = log_domain ? lu.as<double>() : u.as<double>();
  const double* pv = log_domain ? lv.as<double>() : v.as<double>();
  if (dk.dense) {
    KDense kf{dk.K.as<double>(), dk.n};
    if (log_domain) dense_readout_t<true>(ctx, kf, dk, pu, pv, a, b, want_objective, uot, lambda, eps, out, rmh, cmh);
    else dense_readout_t<false>(ctx, kf, dk, pu, pv, a, b, want_objective, uot, lambda, eps, out, rmh, cmh);
  } else {
    KCoords kf = kcoords_of(dk);
    if (log_domain) dense_readout_t<true>(ctx, kf, dk, pu, pv, a, b, want_objective, uot, lambda, eps, out, rmh, cmh);
    else dense_readout_t<false>(ctx, kf, dk, pu, pv, a, b, want_objective, uot, lambda, eps, out, rmh, cmh);
  }
}

}  // namespace spk
