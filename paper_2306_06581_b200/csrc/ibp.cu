// ibp.cu -- Spar-IBP barycenters on the device.
//
// Reference: ibp<Kernel> (include/sparsink/barycenter.hpp:48-206) and
// spar_ibp (proj/src/barycenter.cpp:8-40): sketch every K_k with the
// column-constant plan (barycenter_probabilities, sparsify.cpp:117-135) and
// seed mix_seed(seed, k), then iterate, for every k with w_k > 0,
//   v_k = b_k / K_k' u_k            (column pass over the CSC mirror)
//   kv_k = K_k v_k                   (row pass over the CSR)
// then q = prod_k kv_k^{w_k}, u_k = q / kv_k, stop on ||q - q_prev||_1 <= delta.
// Kernels run one thread per output summing in the reference's index order
// without FMA, so q matches the CPU reference to pow()'s ULPs. Masks and
// guards follow the reference (Mask / Error policies, divergence restore).
// The iteration is host-driven (a flag read per pass): barycenter problems
// are small (grids of 10^2..10^4 atoms) and this keeps the reference's
// sequential "first failing index" semantics.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace spk {
namespace ibp {

constexpr unsigned long long kNone = ~0ull;

struct Flags {
  unsigned long long bad;   // first failing index of the pass (kNone = none)
  unsigned long long masked;  // newly masked rows
};

template <class VT>
__global__ void col_kernel(int64_t n, const long long* ptr, const uint32_t* idx, const VT* val, const double* u,
                           const double* b, unsigned char* col_ok, double* v, int policy, Flags* f) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    if (!col_ok[j]) {
      v[j] = 0.0;
      continue;
    }
    double tmp = 0.0;  // spmv_t: rows ascending, skipping u_i == 0 (sparsify.cpp:215-226)
    for (long long p = ptr[j]; p < ptr[j + 1]; ++p) {
      const double ui = u[idx[p]];
      if (ui == 0.0) continue;
      tmp = dadd(tmp, dmul((double)val[p], ui));
    }
    if (tmp <= 0.0 || !isfinite(tmp)) {
      if (policy == SPK_POLICY_MASK && tmp == 0.0) {  // barycenter.hpp:125-130
        col_ok[j] = 0;
        v[j] = 0.0;
        continue;
      }
      atomicMin(&f->bad, (unsigned long long)j);
      continue;
    }
    const double vj = b[j] / tmp;
    v[j] = vj;
    if (!(vj <= 1e150) && policy == SPK_POLICY_MASK) atomicMin(&f->bad, (unsigned long long)j);
  }
}

template <class VT>
__global__ void row_kernel(int64_t n, const long long* ptr, const uint32_t* idx, const VT* val, const double* v,
                           unsigned char* row_ok, double* q, double* kv, int policy, Flags* f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;  // spmv: columns ascending (sparsify.cpp:203-213)
    for (long long p = ptr[i]; p < ptr[i + 1]; ++p) acc = dadd(acc, dmul((double)val[p], v[idx[p]]));
    kv[i] = acc;
    if (!row_ok[i]) continue;
    if (acc <= 0.0 || !isfinite(acc)) {
      if (policy == SPK_POLICY_MASK && acc == 0.0) {  // barycenter.hpp:147-152
        row_ok[i] = 0;
        q[i] = 0.0;
        atomicAdd(&f->masked, 1ull);
        continue;
      }
      atomicMin(&f->bad, (unsigned long long)i);
    }
  }
}

// q_i = prod_k kv_k(i)^{w_k} over active kernels, in k order (barycenter.hpp:170-181)
__global__ void q_kernel(int64_t n, int m, const double* w, const double* kv, const unsigned char* row_ok, double* q,
                         int policy, Flags* f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!row_ok[i]) continue;
    double acc = 1.0;
    for (int k = 0; k < m; ++k) {
      if (w[k] == 0.0) continue;
      acc = dmul(acc, pow(kv[(int64_t)k * n + i], w[k]));
    }
    if (!(acc <= 1e150) && policy == SPK_POLICY_MASK) atomicMin(&f->bad, (unsigned long long)i);
    q[i] = acc;
  }
}

__global__ void u_kernel(int64_t n, int m, const double* w, const double* kv, const unsigned char* row_ok,
                         const double* q, double* u, int policy, Flags* f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int k = 0; k < m; ++k) {
      if (w[k] == 0.0) continue;
      const double uk = row_ok[i] ? q[i] / kv[(int64_t)k * n + i] : 0.0;
      u[(int64_t)k * n + i] = uk;
      if (!(uk <= 1e150) && policy == SPK_POLICY_MASK) atomicMin(&f->bad, (unsigned long long)i);
    }
  }
}

// ||q - q_prev||_1 in index order (barycenter.hpp:195-197)
__global__ void err_kernel(int64_t n, const double* q, const double* qp, double* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double e = 0.0;
  for (int64_t i = 0; i < n; ++i) e = dadd(e, fabs(dsub(q[i], qp[i])));
  *out = e;
}

__global__ void init_kernel(int64_t n, int m, const unsigned char* row_ok, double* q, double* u, double* v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    q[i] = row_ok[i] ? 1.0 / (double)n : 0.0;
    for (int k = 0; k < m; ++k) {
      u[(int64_t)k * n + i] = 1.0;
      v[(int64_t)k * n + i] = 1.0;
    }
  }
}

__global__ void cover_kernel(int64_t n, const long long* row_ptr, const long long* col_ptr, unsigned char* row_ok,
                             unsigned char* col_ok) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    row_ok[i] = row_ok[i] && row_ptr[i + 1] > row_ptr[i];
    col_ok[i] = col_ptr[i + 1] > col_ptr[i];
  }
}

__global__ void fill_u8(unsigned char* p, int64_t n, unsigned char v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void reset_flags(Flags* f) {
  f->bad = kNone;
  f->masked = 0;
}

int grid(spk_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 127) / 128, (int64_t)ctx->num_sms * 8));
}

struct Out {
  int64_t iterations = 0;
  int converged = 0, diverged = 0;
  int64_t masked = 0;
};

// ibp<SparseKernel> (barycenter.hpp:48-206) on device sketches.
void run(spk_ctx* ctx, spk_sketch* const* sks, int m, const double* b_host, const double* w_host, double delta,
         int64_t max_iter, int policy, double* q_host, Out& out) {
  if (m <= 0) fail(SPK_E_LENGTH_MISMATCH, "empty barycenter problem");
  double wsum = 0.0;
  for (int k = 0; k < m; ++k) {
    if (w_host[k] < 0.0) fail(SPK_E_NEGATIVE_WEIGHT, "barycenter weight");
    wsum += w_host[k];
  }
  if (std::abs(wsum - 1.0) > 1e-10) fail(SPK_E_NOT_NORMALIZED, "barycenter weights must sum to 1");
  const int64_t n = sks[0]->n;
  for (int k = 0; k < m; ++k)
    if (sks[k]->n != n) fail(SPK_E_LENGTH_MISMATCH, "all measures must share one dimension");
  cudaStream_t s = ctx->stream;
  DBuf w(sizeof(double) * m), b(sizeof(double) * m * n), q(sizeof(double) * n), qp(sizeof(double) * n),
      u(sizeof(double) * m * n), v(sizeof(double) * m * n), kv(sizeof(double) * m * n), row_ok(n), col_ok(m * n),
      flags(sizeof(Flags)), err(sizeof(double));
  upload(ctx, w, w_host, sizeof(double) * m);
  upload(ctx, b, b_host, sizeof(double) * m * n);
  SPK_CUDA(cudaMemsetAsync(kv.p, 0, kv.bytes, s));
  fill_u8<<<grid(ctx, n), 128, 0, s>>>(row_ok.as<unsigned char>(), n, 1);
  SPK_CUDA(cudaMemsetAsync(col_ok.p, 0, col_ok.bytes, s));
  ++ctx->launches;
  // coverage: a row survives only if every active kernel reaches it (:76-85)
  for (int k = 0; k < m; ++k) {
    if (w_host[k] == 0.0) continue;
    cover_kernel<<<grid(ctx, n), 128, 0, s>>>(n, sks[k]->row_ptr.as<long long>(), sks[k]->col_ptr.as<long long>(),
                                              row_ok.as<unsigned char>(), col_ok.as<unsigned char>() + k * n);
    ++ctx->launches;
  }
  std::vector<unsigned char> hr(n), hc(m * n);
  download(ctx, hr.data(), row_ok, n);
  download(ctx, hc.data(), col_ok, m * n);
  int64_t masked = 0;
  for (int64_t i = 0; i < n; ++i) masked += hr[i] ? 0 : 1;
  bool col_gap = false;
  for (int k = 0; k < m; ++k)
    if (w_host[k] != 0.0)
      for (int64_t j = 0; j < n; ++j) col_gap = col_gap || !hc[k * n + j];
  if ((masked > 0 || col_gap) && policy == SPK_POLICY_ERROR)
    fail(SPK_E_ZERO_DENOMINATOR, "a kernel has empty rows or columns");
  if (masked == n) fail(SPK_E_DEGENERATE_SKETCH_ERROR, "no atom covered by all kernels");
  init_kernel<<<grid(ctx, n), 128, 0, s>>>(n, m, row_ok.as<unsigned char>(), q.as<double>(), u.as<double>(),
                                           v.as<double>());
  ++ctx->launches;

  Flags fl;
  auto pass_flags = [&]() {
    download(ctx, &fl, flags, sizeof fl);
    masked += (int64_t)fl.masked;
    return fl.bad;
  };
  bool converged = false, diverged = false;
  int64_t t = 0;
  while (t < max_iter) {
    ++t;
    SPK_CUDA(cudaMemcpyAsync(qp.p, q.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    for (int k = 0; k < m && !diverged; ++k) {
      if (w_host[k] == 0.0) continue;
      spk_sketch* sk = sks[k];
      const bool f32 = sk->value_type == SPK_VALUES_F32;
      reset_flags<<<1, 1, 0, s>>>(flags.as<Flags>());
      if (f32)
        col_kernel<float><<<grid(ctx, n), 128, 0, s>>>(n, sk->col_ptr.as<long long>(), sk->row_idx.as<uint32_t>(),
                                                       sk->values_t.as<float>(), u.as<double>() + k * n,
                                                       b.as<double>() + k * n, col_ok.as<unsigned char>() + k * n,
                                                       v.as<double>() + k * n, policy, flags.as<Flags>());
      else
        col_kernel<double><<<grid(ctx, n), 128, 0, s>>>(n, sk->col_ptr.as<long long>(), sk->row_idx.as<uint32_t>(),
                                                        sk->values_t.as<double>(), u.as<double>() + k * n,
                                                        b.as<double>() + k * n, col_ok.as<unsigned char>() + k * n,
                                                        v.as<double>() + k * n, policy, flags.as<Flags>());
      ctx->launches += 2;
      if (pass_flags() != kNone) {
        if (policy == SPK_POLICY_MASK) {
          diverged = true;
          break;
        }
        fail(SPK_E_ZERO_DENOMINATOR, "K'u underflowed in IBP");
      }
      reset_flags<<<1, 1, 0, s>>>(flags.as<Flags>());
      if (f32)
        row_kernel<float><<<grid(ctx, n), 128, 0, s>>>(n, sk->row_ptr.as<long long>(), sk->col_idx.as<uint32_t>(),
                                                       sk->values.as<float>(), v.as<double>() + k * n,
                                                       row_ok.as<unsigned char>(), q.as<double>(),
                                                       kv.as<double>() + k * n, policy, flags.as<Flags>());
      else
        row_kernel<double><<<grid(ctx, n), 128, 0, s>>>(n, sk->row_ptr.as<long long>(), sk->col_idx.as<uint32_t>(),
                                                        sk->values.as<double>(), v.as<double>() + k * n,
                                                        row_ok.as<unsigned char>(), q.as<double>(),
                                                        kv.as<double>() + k * n, policy, flags.as<Flags>());
      ctx->launches += 2;
      if (pass_flags() != kNone) {
        if (policy == SPK_POLICY_MASK) {
          diverged = true;
          break;
        }
        fail(SPK_E_ZERO_DENOMINATOR, "Kv underflowed in IBP");
      }
    }
    if (diverged) {  // keep the last iterate (:160-163)
      SPK_CUDA(cudaMemcpyAsync(q.p, qp.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      break;
    }
    if (masked == n) fail(SPK_E_DEGENERATE_SKETCH_ERROR, "masking removed every atom");
    reset_flags<<<1, 1, 0, s>>>(flags.as<Flags>());
    q_kernel<<<grid(ctx, n), 128, 0, s>>>(n, m, w.as<double>(), kv.as<double>(), row_ok.as<unsigned char>(),
                                          q.as<double>(), policy, flags.as<Flags>());
    u_kernel<<<grid(ctx, n), 128, 0, s>>>(n, m, w.as<double>(), kv.as<double>(), row_ok.as<unsigned char>(),
                                          q.as<double>(), u.as<double>(), policy, flags.as<Flags>());
    err_kernel<<<1, 1, 0, s>>>(n, q.as<double>(), qp.as<double>(), err.as<double>());
    ctx->launches += 4;
    if (pass_flags() != kNone) {
      diverged = true;
      SPK_CUDA(cudaMemcpyAsync(q.p, qp.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      break;
    }
    double e = 0.0;
    download(ctx, &e, err, sizeof e);
    if (e <= delta) {
      converged = true;
      break;
    }
  }
  download(ctx, q_host, q, sizeof(double) * n);
  out.iterations = t;
  out.converged = converged ? 1 : 0;
  out.diverged = diverged ? 1 : 0;
  out.masked = masked;
}

}  // namespace ibp
}  // namespace spk

using namespace spk;

namespace {
void fill_report(spk_ibp_report* rep, const ibp::Out& o, double secs) {
  if (!rep) return;
  rep->iterations = o.iterations;
  rep->converged = o.converged;
  rep->diverged = o.diverged;
  rep->masked_atoms = o.masked;
  rep->wall_time_s = secs;
}
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

extern "C" {

int spk_ibp(spk_ctx* ctx, spk_sketch* const* sketches, int32_t m, const double* b, const double* w, double delta,
            int64_t max_iter, int32_t policy, double* q, spk_ibp_report* rep) {
  if (!ctx || !sketches || !q) return SPK_STATUS_INPUT;
  return guard(ctx, [&] {
    const double t0 = now_s();
    ibp::Out o;
    ibp::run(ctx, sketches, m, b, w, delta, max_iter, policy, q, o);
    fill_report(rep, o, now_s() - t0);
  });
}

int spk_spar_ibp(spk_ctx* ctx, const spk_kernel_desc* kds, int32_t m, const double* b, const double* w, double delta,
                 int64_t max_iter, double s, uint64_t seed, int32_t strict, int32_t value_type, double* q,
                 spk_ibp_report* rep) {
  if (!ctx || !kds || !q) return SPK_STATUS_INPUT;
  return guard(ctx, [&] {
    const double t0 = now_s();
    if (m <= 0) fail(SPK_E_LENGTH_MISMATCH, "kernels, measures and weights must align");
    const int64_t n = kds[0].n;
    std::vector<std::unique_ptr<spk_sketch>> sks;
    std::vector<spk_sketch*> ptrs;
    for (int k = 0; k < m; ++k) {
      if (kds[k].n != n) fail(SPK_E_LENGTH_MISMATCH, "all measures must share one dimension");
      DevKernel dk;
      make_dev_kernel(ctx, &kds[k], kds[k].kernel_epsilon > 0 ? kds[k].kernel_epsilon : 1.0, dk, false);
      PlanInfo plan;  // barycenter_probabilities (sparsify.cpp:117-135): rows 1/n, columns sqrt(b_k)
      build_plan(ctx, dk, b + (int64_t)k * n, b + (int64_t)k * n, SPK_PLAN_BARYCENTER, INFINITY, dk.eps, 0.0, plan);
      auto sk = std::make_unique<spk_sketch>();
      sk->ctx = ctx;
      sk->device = ctx->device;
      sample_sketch(ctx, dk, plan, s, mix_seed(seed, (uint64_t)k), value_type, sk.get());
      if (strict) {  // barycenter.cpp:26-32
        std::vector<long long> rp(n + 1), cp(n + 1);
        download(ctx, rp.data(), sk->row_ptr, sizeof(long long) * (n + 1));
        download(ctx, cp.data(), sk->col_ptr, sizeof(long long) * (n + 1));
        for (int64_t i = 0; i < n; ++i)
          if (rp[i + 1] == rp[i] || cp[i + 1] == cp[i])
            fail(SPK_E_DEGENERATE_SKETCH_ERROR,
                 "sketch " + std::to_string(k) + " orphaned atom " + std::to_string(i));
      }
      ptrs.push_back(sk.get());
      sks.push_back(std::move(sk));
    }
    ibp::Out o;
    ibp::run(ctx, ptrs.data(), m, b, w, delta, max_iter, strict ? SPK_POLICY_ERROR : SPK_POLICY_MASK, q, o);
    fill_report(rep, o, now_s() - t0);
  });
}

}  // extern "C"
