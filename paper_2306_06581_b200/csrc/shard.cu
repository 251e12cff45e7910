// shard.cu -- row/column-sharded Spar-Sink for one process per GPU
// (north-star "rows of K~ are sharded across the 8 GPUs").
//
// Partition: rank r owns atoms [r*m, min(n,(r+1)*m)), m = ceil(n/W), as rows
// (CSR sampled locally: poisson_sparsify row streams, sparsify.cpp:184-198,
// so the union over ranks is the single-GPU sketch bit for bit) and as
// columns (CSC assembled once from every rank's row slab by an all-to-all).
//
// Scaling vectors live in a "gathered" layout: W blocks of stride m + T
// doubles (T = SPK_SHARD_TAIL), block r = rank r's slab then its tail. The
// sketch's column indices (CSR) and row indices (CSC) are remapped into that
// layout once, so a half-step reads the gathered vector directly and one
// all-gather per half (issued by the caller) completes it. The tail carries
// the slab's residual partial, dynamic-mask count and first failing index,
// so every rank re-derives the loop decisions of detail::scaling_loop
// (solvers.hpp:284-364) from the same gathered bits -- identical decisions,
// no host round trip per iteration.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <string>

#include "common.cuh"
#include "internal.h"
#include "ksrc.cuh"
#include "loop_core.cuh"
#include "rowdot.cuh"
#include "shard_core.cuh"

namespace spk {
namespace shard {

template <bool LOG, class VT>
__global__ void __launch_bounds__(kThreads) half_kernel(HalfArgs A) {
  __shared__ State S;
  if (threadIdx.x == 0) {
    S = *A.st_in;
    decide<LOG>(A, S);
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) *A.st_out = S;
  if (S.stopped || !A.compute) return;

  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const VT* val = static_cast<const VT*>(A.val);
  double err = 0.0;
  long long masks = 0;
  for (int64_t i = warp; i < A.m_own; i += nw) {
    if (!A.ne[i]) {
      if (lane == 0) A.out[i] = __ldcg(A.old + i);
      continue;
    }
    const double tmp = row_apply<LOG, false, VT>(val, A.idx, __ldg(A.ptr + i), __ldg(A.ptr + i + 1), A.x, lane);
    if (lane == 0)
      err += loopcore::finalize_atom<LOG>(i, tmp, __ldcg(A.old + i), __ldg(A.w + i), A.exponent, A.policy, (int)A.t,
                                          A.ne, A.dyn, A.out, A.flag, masks);
  }
  finish_half(A, err, masks);
}

// j (global) -> position in the gathered layout
__global__ void remap_kernel(uint32_t* idx, int64_t cnt, uint32_t m) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnt; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t j = idx[k];
    idx[k] = j + (j / m) * (uint32_t)kT;
  }
}

__global__ void export_counts_kernel(const long long* col_ptr, int64_t n, int64_t m, int world, long long* counts) {
  const int64_t total = (int64_t)world * m;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x)
    counts[k] = k < n ? col_ptr[k + 1] - col_ptr[k] : 0;
}

__global__ void export_sizes_kernel(const long long* col_ptr, int64_t n, int64_t m, int world, long long* sizes) {
  const int d = threadIdx.x;
  if (d >= world) return;
  const int64_t a0 = (int64_t)d * m, a1 = (int64_t)(d + 1) * m;
  const int64_t c0 = a0 < n ? a0 : n, c1 = a1 < n ? a1 : n;
  sizes[d] = col_ptr[c1] - col_ptr[c0];
}

__global__ void add_base_kernel(const uint32_t* in, int64_t cnt, uint32_t base, uint32_t* out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnt; k += (int64_t)gridDim.x * blockDim.x)
    out[k] = in[k] + base;
}

__global__ void col_totals_kernel(const long long* counts, int64_t m, int64_t m_own, int world, long long* tot) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m_own; c += (int64_t)gridDim.x * blockDim.x) {
    long long s = 0;
    for (int r = 0; r < world; ++r) s += counts[(int64_t)r * m + c];
    tot[c] = s;
  }
}

// One warp per owned column: sources in rank order (rows ascending across
// ranks, and inside each source already ascending).
template <class VT>
__global__ void import_kernel(const long long* counts, const long long* src_off, const long long* col_ptr,
                              int64_t m, int64_t m_own, int world, const uint32_t* rows, const VT* vals,
                              uint32_t* row_idx, VT* vals_t) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t mm = (uint32_t)m;
  for (int64_t c = warp; c < m_own; c += nw) {
    long long dst = col_ptr[c];
    for (int r = 0; r < world; ++r) {
      const long long cnt = counts[(int64_t)r * m + c], src = src_off[(int64_t)r * m + c];
      for (long long k = lane; k < cnt; k += 32) {
        const uint32_t i = rows[src + k];
        row_idx[dst + k] = i + (i / mm) * (uint32_t)kT;
        vals_t[dst + k] = vals[src + k];
      }
      dst += cnt;
    }
  }
}

__global__ void coverage_kernel(const long long* row_ptr, const long long* col_ptr, int64_t m_own,
                                unsigned char* row_ne, unsigned char* col_ne, unsigned long long* empty) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m_own; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned char r = row_ptr[i + 1] > row_ptr[i];
    const unsigned char c = col_ptr[i + 1] > col_ptr[i];
    row_ne[i] = r;
    col_ne[i] = c;
    if (!r) atomicAdd(&empty[0], 1ull);
    if (!c) atomicAdd(&empty[1], 1ull);
  }
}

template <bool LOG>
__global__ void init_block_kernel(int64_t m, int64_t m_own, const unsigned char* row_ne, const unsigned char* col_ne,
                                  double* u, double* v) {
  const double on = LOG ? 0.0 : 1.0;
  const double off = LOG ? -CUDART_INF : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m + kT; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < m_own) {
      u[i] = row_ne[i] ? on : off;
      v[i] = col_ne[i] ? on : off;
    } else {
      u[i] = 0.0;  // slab padding and the tail
      v[i] = 0.0;
    }
  }
}

__global__ void log_kernel(int64_t n, const double* a, double* la) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    la[i] = a[i] > 0.0 ? log(a[i]) : -CUDART_INF;
}

__global__ void state_init_kernel(State* st, long long mr, long long mc) {
  State s{};
  s.masked_rows = mr;
  s.masked_cols = mc;
  st[0] = s;
  st[1] = s;
}

__global__ void reset_kernel(unsigned int* ticket, unsigned long long* flag) {
  *ticket = 0u;
  *flag = kNone;
}

// ---- readout ----
template <bool LOG>
__device__ __forceinline__ double plan_entry(double ui, double k, double vj) {
  if (LOG) {
    if (ui == -CUDART_INF || vj == -CUDART_INF) return 0.0;
    return exp(dadd(dadd(ui, log(k)), vj));
  }
  return dmul(dmul(ui, k), vj);
}

template <bool LOG, bool OBJ, class VT>
__global__ void read_rows_kernel(int64_t m_own, int64_t base, int64_t stride, const long long* ptr,
                                 const uint32_t* idx, const VT* val, const double* u_own, const double* v, CostSrc cs,
                                 double* row_m, double* row_c, double* row_h, unsigned long long* inf_flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < m_own; i += nw) {
    double mm = 0.0, c = 0.0, h = 0.0;
    const double ui = u_own[i];
    for (long long p = ptr[i] + lane; p < ptr[i + 1]; p += 32) {
      const int64_t jj = idx[p];
      const double t = plan_entry<LOG>(ui, (double)val[p], v[jj]);
      if (!(t > 0.0)) continue;
      mm += t;
      if (OBJ) {
        const int64_t j = jj - (jj / stride) * kT;
        const double cij = cs(base + i, j);
        if (isinf(cij)) atomicMin(inf_flag, (unsigned long long)(base + i));
        c = dadd(c, dmul(t, cij));
        h = dsub(h, dmul(t, dsub(log(t), 1.0)));
      }
    }
    mm = warp_sum(mm);
    if (OBJ) {
      c = warp_sum(c);
      h = warp_sum(h);
    }
    if (lane == 0) {
      row_m[i] = mm;
      if (OBJ) {
        row_c[i] = c;
        row_h[i] = h;
      }
    }
  }
}

template <bool LOG, class VT>
__global__ void read_cols_kernel(int64_t m_own, const long long* ptr, const uint32_t* idx, const VT* val,
                                 const double* u, const double* v_own, double* col_m) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp; c < m_own; c += nw) {
    double mm = 0.0;
    const double vj = v_own[c];
    for (long long p = ptr[c] + lane; p < ptr[c + 1]; p += 32) {
      const double t = plan_entry<LOG>(u[idx[p]], (double)val[p], vj);
      if (t > 0.0) mm += t;
    }
    mm = warp_sum(mm);
    if (lane == 0) col_m[c] = mm;
  }
}

__device__ __forceinline__ double kl_term(double x, double y, int64_t gi, unsigned long long* bad) {
  if (x > 0.0) {  // kl_divergence (solvers.cpp:250-257)
    if (y <= 0.0) atomicMin(bad, (unsigned long long)gi);
    return dadd(dsub(dmul(x, log(x / y)), x), y);
  }
  return y;
}

// One block: the slab's sums in a fixed order (deterministic per rank).
__global__ void read_sums_kernel(int64_t m_own, int64_t base, const double* row_m, const double* col_m,
                                 const double* row_c, const double* row_h, const double* a, const double* b, int obj,
                                 int uot, unsigned long long* bad, double* out) {
  __shared__ double sm[6][32];
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int64_t per = (m_own + blockDim.x - 1) / blockDim.x;
  const int64_t lo = threadIdx.x * per, hi = lo + per < m_own ? lo + per : m_own;
  for (int64_t i = lo; i < hi; ++i) {
    acc[0] += fabs(dsub(row_m[i], a[i]));
    acc[1] += fabs(dsub(col_m[i], b[i]));
    if (obj) {
      acc[2] += row_c[i];
      acc[3] += row_h[i];
      if (uot) {
        acc[4] += kl_term(row_m[i], a[i], base + i, bad);
        acc[5] += kl_term(col_m[i], b[i], base + i, bad + 1);
      }
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const double s = warp_sum(acc[q]);
    if (lane == 0) sm[q][w] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < 6; ++q) {
      double s = 0.0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += sm[q][k];
      out[q] = s;
    }
  }
}

__global__ void fill3_kernel(unsigned long long* p) {
  p[0] = kNone;
  p[1] = kNone;
  p[2] = kNone;
}

int grid_rows(spk_ctx* ctx, int64_t rows) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((rows + 15) / 16, (int64_t)ctx->num_sms * 4));
}
int grid_elems(spk_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8));
}

}  // namespace shard
}  // namespace spk

struct spk_shard {
  spk_ctx* ctx = nullptr;
  int device = 0;
  int world = 1, rank = 0;
  int64_t n = 0, m = 0, stride = 0, lo = 0, hi = 0, m_own = 0;
  spk::DevKernel dk;
  spk_sketch rows;  // CSR of the row slab (columns remapped) + its by-column copy for export
  int value_type = SPK_VALUES_F64;
  size_t vbytes = 8;
  spk::DBuf col_ptr, row_idx, vals_t;  // CSC of the column slab (rows remapped)
  int64_t col_nnz = 0;
  bool imported = false;
  spk::DBuf a, b, la, lb;  // own slabs
  double a_total = 0.0, b_total = 0.0;
  spk::DBuf row_ne, col_ne, dyn_row, dyn_col;
  long long empty_rows = -1, empty_cols = -1;
  spk::DBuf state, part, ticket, flag;
  int part_cap = 0;
  long long calls = 0;  // half/finish launches since begin (selects the state buffer)
  bool began = false;
  int log_domain = 0, policy = SPK_POLICY_MASK;
  double exponent = 1.0, delta = 0.0;
  long long max_iter = 0;
  double kernel_mean_part = 0.0;
  int64_t kernel_nnz = 0;
  int factorized = 0;
  spk::DBuf rd_row_m, rd_col_m, rd_row_c, rd_row_h, rd_flags, rd_out;
  spk::shard::BlockedShard blk;  // slab x block layouts of both halves (fast linear loop)
  bool blk_tried = false;
};

using namespace spk;

namespace {

void slab_bounds(int64_t n, int world, int rank, int64_t& m, int64_t& lo, int64_t& hi) {
  if (world < 1 || rank < 0 || rank >= world) fail(SPK_E_LENGTH_MISMATCH, "bad shard rank / world");
  m = (n + world - 1) / world;
  lo = std::min<int64_t>(n, (int64_t)rank * m);
  hi = std::min<int64_t>(n, lo + m);
}

void need_coords(const spk_kernel_desc* kd) {
  if (!kd) fail(SPK_E_LENGTH_MISMATCH, "null kernel descriptor");
  if (kd->K || !kd->x) fail(SPK_E_DIMENSION_MISMATCH, "sharded solves need the coordinate form");
}

template <bool LOG, class VT>
void launch_half(spk_shard* sh, shard::HalfArgs& A, int grid) {
  shard::half_kernel<LOG, VT><<<grid, shard::kThreads, 0, sh->ctx->stream>>>(A);
}

}  // namespace

namespace spk {
void shard_set_calls(spk_shard* sh, long long calls) { sh->calls = calls; }
}  // namespace spk

extern "C" {

int spk_shard_plan_rows(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b, int plan_kind,
                        double lambda, double epsilon, int32_t world, int32_t rank, double* row_sum_dev,
                        int64_t* row_nnz_dev, int32_t* needs_pass) {
  if (!ctx) return SPK_STATUS_INPUT;
  return guard(ctx, [&] {
    need_coords(kd);
    DevKernel dk;
    make_dev_kernel(ctx, kd, epsilon, dk, false);
    int64_t m, lo, hi;
    slab_bounds(dk.n, world, rank, m, lo, hi);
    PlanInfo plan;
    const bool need = plan_weights(ctx, dk, a, b, plan_kind, lambda, epsilon, plan);
    if (needs_pass) *needs_pass = need ? 1 : 0;
    if (need) plan_pass_rows(ctx, dk, plan, lo, hi, reinterpret_cast<long long*>(row_nnz_dev), row_sum_dev);
    SPK_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int spk_shard_create(spk_ctx* ctx, const spk_kernel_desc* kd, const double* a, const double* b, int plan_kind,
                     double lambda, double epsilon, double s, uint64_t seed, const spk_sketch_opts* opts,
                     int32_t world, int32_t rank, const double* row_sum_all_dev, const int64_t* row_nnz_all_dev,
                     spk_shard** out) {
  if (!ctx || !out) return SPK_STATUS_INPUT;
  *out = nullptr;
  return guard(ctx, [&] {
    need_coords(kd);
    spk_sketch_opts o{};
    if (opts) o = *opts;
    auto sh = std::make_unique<spk_shard>();
    sh->ctx = ctx;
    sh->device = ctx->device;
    sh->world = world;
    sh->rank = rank;
    make_dev_kernel(ctx, kd, epsilon, sh->dk, /*need_cost=*/true);
    const int64_t n = sh->dk.n;
    sh->n = n;
    slab_bounds(n, world, rank, sh->m, sh->lo, sh->hi);
    sh->m_own = sh->hi - sh->lo;
    sh->stride = sh->m + shard::kT;
    if ((double)world * (double)sh->stride > 4294967295.0) fail(SPK_E_BUDGET_TOO_LARGE, "n too large for u32 indices");
    PlanInfo plan;
    const bool need = plan_weights(ctx, sh->dk, a, b, plan_kind, lambda, epsilon, plan);
    if (need) {
      if (!row_sum_all_dev || !row_nnz_all_dev) fail(SPK_E_LENGTH_MISMATCH, "plan needs the gathered row sums");
      plan.d_row_nnz.alloc(sizeof(long long) * n);
      plan.d_row_sum.alloc(sizeof(double) * n);
      plan.have_rows = true;
      SPK_CUDA(cudaMemcpyAsync(plan.d_row_nnz.p, row_nnz_all_dev, sizeof(long long) * n, cudaMemcpyDeviceToDevice,
                               ctx->stream));
      SPK_CUDA(cudaMemcpyAsync(plan.d_row_sum.p, row_sum_all_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                               ctx->stream));
    }
    plan_finish(ctx, sh->dk, need, o.theta > 0.0 ? o.theta : 0.0, plan);
    spk_sketch& R = sh->rows;
    R.ctx = ctx;
    R.device = ctx->device;
    sample_sketch(ctx, sh->dk, plan, s, seed, o.value_type, &R, sh->lo, sh->hi);
    sh->value_type = o.value_type;
    sh->vbytes = o.value_type == SPK_VALUES_F32 ? 4 : 8;
    sh->kernel_mean_part = R.kernel_mean;
    sh->kernel_nnz = plan.kernel_nnz;
    sh->factorized = plan.factorized ? 1 : 0;
    if (R.nnz > 0)
      shard::remap_kernel<<<shard::grid_elems(ctx, R.nnz), 256, 0, ctx->stream>>>(R.col_idx.as<uint32_t>(), R.nnz,
                                                                                 (uint32_t)sh->m);
    ++ctx->launches;
    upload(ctx, sh->a, a + sh->lo, sizeof(double) * std::max<int64_t>(sh->m_own, 1));
    upload(ctx, sh->b, b + sh->lo, sizeof(double) * std::max<int64_t>(sh->m_own, 1));
    sh->a_total = seq_total(a, n);
    sh->b_total = seq_total(b, n);
    SPK_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = sh.release();
  });
}

void spk_shard_free(spk_shard* sh) {
  if (!sh) return;
  cudaSetDevice(sh->device);
  cudaDeviceSynchronize();  // as spk_sketch_free: the buffers return to the pool once idle
  {
    AllocStreamScope scope(nullptr);
    delete sh;
  }
  (void)cudaGetLastError();
}

int spk_shard_info(const spk_shard* sh, int64_t* n, int64_t* m, int64_t* stride, int64_t* lo, int64_t* hi,
                   int64_t* row_nnz, int64_t* col_nnz, int32_t* value_bytes, double* kernel_mean_part,
                   int64_t* kernel_nnz, int32_t* factorized_plan) {
  if (!sh) return SPK_STATUS_INPUT;
  if (n) *n = sh->n;
  if (m) *m = sh->m;
  if (stride) *stride = sh->stride;
  if (lo) *lo = sh->lo;
  if (hi) *hi = sh->hi;
  if (row_nnz) *row_nnz = sh->rows.nnz;
  if (col_nnz) *col_nnz = sh->imported ? sh->col_nnz : -1;
  if (value_bytes) *value_bytes = (int32_t)sh->vbytes;
  if (kernel_mean_part) *kernel_mean_part = sh->kernel_mean_part;
  if (kernel_nnz) *kernel_nnz = sh->kernel_nnz;
  if (factorized_plan) *factorized_plan = sh->factorized;
  return SPK_OK;
}

int spk_shard_export(spk_shard* sh, int64_t* counts_dev, uint32_t* rows_dev, void* vals_dev, int64_t* send_sizes) {
  if (!sh) return SPK_STATUS_INPUT;
  return guard(sh->ctx, [&] {
    spk_ctx* ctx = sh->ctx;
    spk_sketch& R = sh->rows;
    if (!R.col_ptr.p) fail(SPK_E_LENGTH_MISMATCH, "row slab already exported");
    shard::export_counts_kernel<<<shard::grid_elems(ctx, sh->world * sh->m), 256, 0, ctx->stream>>>(
        R.col_ptr.as<long long>(), sh->n, sh->m, sh->world, reinterpret_cast<long long*>(counts_dev));
    DBuf sizes(sizeof(long long) * sh->world);
    shard::export_sizes_kernel<<<1, 1024, 0, ctx->stream>>>(R.col_ptr.as<long long>(), sh->n, sh->m, sh->world,
                                                             sizes.as<long long>());
    ctx->launches += 2;
    if (R.nnz > 0) {
      shard::add_base_kernel<<<shard::grid_elems(ctx, R.nnz), 256, 0, ctx->stream>>>(
          R.row_idx.as<uint32_t>(), R.nnz, (uint32_t)sh->lo, rows_dev);
      ++ctx->launches;
      SPK_CUDA(cudaMemcpyAsync(vals_dev, R.values_t.p, sh->vbytes * R.nnz, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    download(ctx, send_sizes, sizes, sizeof(long long) * sh->world);
  });
}

int spk_shard_import(spk_shard* sh, const int64_t* recv_counts_dev, const uint32_t* recv_rows_dev,
                     const void* recv_vals_dev, int64_t total) {
  if (!sh) return SPK_STATUS_INPUT;
  return guard(sh->ctx, [&] {
    spk_ctx* ctx = sh->ctx;
    const int64_t W = sh->world, m = sh->m, mo = sh->m_own;
    const long long* counts = reinterpret_cast<const long long*>(recv_counts_dev);
    if (total > 0xffffffffLL) fail(SPK_E_BUDGET_TOO_LARGE, "column slab exceeds 2^32 entries");
    DBuf tot(sizeof(long long) * std::max<int64_t>(mo, 1)), src_off(sizeof(long long) * W * m);
    sh->col_ptr.alloc(sizeof(long long) * (mo + 1));
    SPK_CUDA(cudaMemsetAsync(sh->col_ptr.p, 0, sizeof(long long), ctx->stream));
    if (mo > 0) {
      shard::col_totals_kernel<<<shard::grid_elems(ctx, mo), 256, 0, ctx->stream>>>(counts, m, mo, (int)W,
                                                                                    tot.as<long long>());
      ++ctx->launches;
      size_t tb = 0;
      SPK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, tot.as<long long>(), sh->col_ptr.as<long long>() + 1,
                                             (int)mo, ctx->stream));
      ctx->scratch.ensure(tb);
      SPK_CUDA(cub::DeviceScan::InclusiveSum(ctx->scratch.p, tb, tot.as<long long>(), sh->col_ptr.as<long long>() + 1,
                                             (int)mo, ctx->stream));
    }
    size_t tb = 0;
    SPK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, src_off.as<long long>(), (int)(W * m), ctx->stream));
    ctx->scratch.ensure(tb);
    SPK_CUDA(
        cub::DeviceScan::ExclusiveSum(ctx->scratch.p, tb, counts, src_off.as<long long>(), (int)(W * m), ctx->stream));
    ctx->launches += 2;
    long long got = 0;
    if (mo > 0)
      SPK_CUDA(cudaMemcpyAsync(&got, sh->col_ptr.as<long long>() + mo, sizeof got, cudaMemcpyDeviceToHost,
                               ctx->stream));
    SPK_CUDA(cudaStreamSynchronize(ctx->stream));
    if (got != total) fail(SPK_E_LENGTH_MISMATCH, "column exchange: counts disagree with the entries received");
    sh->col_nnz = total;
    sh->row_idx.alloc(sizeof(uint32_t) * std::max<int64_t>(total, 1));
    sh->vals_t.alloc(sh->vbytes * std::max<int64_t>(total, 1));
    if (mo > 0 && total > 0) {
      if (sh->value_type == SPK_VALUES_F32)
        shard::import_kernel<float><<<shard::grid_rows(ctx, mo), 512, 0, ctx->stream>>>(
            counts, src_off.as<long long>(), sh->col_ptr.as<long long>(), m, mo, (int)W, recv_rows_dev,
            static_cast<const float*>(recv_vals_dev), sh->row_idx.as<uint32_t>(), sh->vals_t.as<float>());
      else
        shard::import_kernel<double><<<shard::grid_rows(ctx, mo), 512, 0, ctx->stream>>>(
            counts, src_off.as<long long>(), sh->col_ptr.as<long long>(), m, mo, (int)W, recv_rows_dev,
            static_cast<const double*>(recv_vals_dev), sh->row_idx.as<uint32_t>(), sh->vals_t.as<double>());
      ++ctx->launches;
    }
    SPK_CUDA(cudaStreamSynchronize(ctx->stream));
    // the row slab's by-column copy has served its purpose
    sh->rows.col_ptr.release();
    sh->rows.row_idx.release();
    sh->rows.values_t.release();
    sh->imported = true;
  });
}

int spk_shard_coverage(spk_shard* sh, int64_t* empty_rows, int64_t* empty_cols) {
  if (!sh) return SPK_STATUS_INPUT;
  return guard(sh->ctx, [&] {
    if (!sh->imported) fail(SPK_E_LENGTH_MISMATCH, "column slab not imported yet");
    spk_ctx* ctx = sh->ctx;
    const int64_t mo = std::max<int64_t>(sh->m_own, 1);
    sh->row_ne.ensure(mo);
    sh->col_ne.ensure(mo);
    DBuf empty(16);
    SPK_CUDA(cudaMemsetAsync(empty.p, 0, 16, ctx->stream));
    if (sh->m_own > 0) {
      shard::coverage_kernel<<<shard::grid_elems(ctx, sh->m_own), 256, 0, ctx->stream>>>(
          sh->rows.row_ptr.as<long long>(), sh->col_ptr.as<long long>(), sh->m_own, sh->row_ne.as<unsigned char>(),
          sh->col_ne.as<unsigned char>(), empty.as<unsigned long long>());
      ++ctx->launches;
    }
    unsigned long long e[2];
    download(ctx, e, empty, sizeof e);
    sh->empty_rows = (long long)e[0];
    sh->empty_cols = (long long)e[1];
    if (empty_rows) *empty_rows = sh->empty_rows;
    if (empty_cols) *empty_cols = sh->empty_cols;
  });
}

int spk_shard_begin(spk_shard* sh, const spk_solver_cfg* cfg, int uot, int policy, int64_t empty_rows_total,
                    int64_t empty_cols_total, double* u0_dev, double* v0_dev) {
  if (!sh || !cfg) return SPK_STATUS_INPUT;
  return guard(sh->ctx, [&] {
    spk_ctx* ctx = sh->ctx;
    if (sh->empty_rows < 0) fail(SPK_E_LENGTH_MISMATCH, "call spk_shard_coverage first");
    if (cfg->max_iter < 0) fail(SPK_E_LENGTH_MISMATCH, "max_iter must be >= 0");
    sh->exponent = solver_exponent(*cfg, uot, sh->a_total, sh->b_total);
    const int64_t n = sh->n;
    // solvers.hpp:269-274 / :411-414
    if ((empty_rows_total || empty_cols_total) && policy == SPK_POLICY_ERROR) {
      if (cfg->stabilize) fail(SPK_E_ZERO_DENOMINATOR, "kernel has empty rows or columns");
      fail(SPK_E_ZERO_DENOMINATOR, "kernel has " + std::to_string(empty_rows_total) + " empty rows and " +
                                       std::to_string(empty_cols_total) + " empty columns");
    }
    if (empty_rows_total == n || empty_cols_total == n)
      fail(SPK_E_DEGENERATE_SKETCH_ERROR, "kernel has no entries at all");
    sh->log_domain = cfg->stabilize ? 1 : 0;
    sh->policy = policy;
    sh->delta = cfg->delta;
    sh->max_iter = cfg->max_iter;
    const int64_t mo = std::max<int64_t>(sh->m_own, 1);
    sh->dyn_row.ensure(sizeof(int) * mo);
    sh->dyn_col.ensure(sizeof(int) * mo);
    SPK_CUDA(cudaMemsetAsync(sh->dyn_row.p, 0, sizeof(int) * mo, ctx->stream));
    SPK_CUDA(cudaMemsetAsync(sh->dyn_col.p, 0, sizeof(int) * mo, ctx->stream));
    // coverage masks are consumed (dynamic masking) by a loop: refresh them
    DBuf empty(16);
    SPK_CUDA(cudaMemsetAsync(empty.p, 0, 16, ctx->stream));
    if (sh->m_own > 0) {
      shard::coverage_kernel<<<shard::grid_elems(ctx, sh->m_own), 256, 0, ctx->stream>>>(
          sh->rows.row_ptr.as<long long>(), sh->col_ptr.as<long long>(), sh->m_own, sh->row_ne.as<unsigned char>(),
          sh->col_ne.as<unsigned char>(), empty.as<unsigned long long>());
      ++ctx->launches;
    }
    if (sh->log_domain) {
      sh->la.ensure(sizeof(double) * mo);
      sh->lb.ensure(sizeof(double) * mo);
      shard::log_kernel<<<shard::grid_elems(ctx, mo), 256, 0, ctx->stream>>>(sh->m_own, sh->a.as<double>(),
                                                                            sh->la.as<double>());
      shard::log_kernel<<<shard::grid_elems(ctx, mo), 256, 0, ctx->stream>>>(sh->m_own, sh->b.as<double>(),
                                                                            sh->lb.as<double>());
      ctx->launches += 2;
    }
    double* u_own = u0_dev + (int64_t)sh->rank * sh->stride;
    double* v_own = v0_dev + (int64_t)sh->rank * sh->stride;
    if (sh->log_domain)
      shard::init_block_kernel<true><<<shard::grid_elems(ctx, sh->stride), 256, 0, ctx->stream>>>(
          sh->m, sh->m_own, sh->row_ne.as<unsigned char>(), sh->col_ne.as<unsigned char>(), u_own, v_own);
    else
      shard::init_block_kernel<false><<<shard::grid_elems(ctx, sh->stride), 256, 0, ctx->stream>>>(
          sh->m, sh->m_own, sh->row_ne.as<unsigned char>(), sh->col_ne.as<unsigned char>(), u_own, v_own);
    sh->state.ensure(2 * sizeof(shard::State));
    sh->ticket.ensure(sizeof(unsigned int));
    sh->flag.ensure(sizeof(unsigned long long));
    const int g = shard::grid_rows(ctx, mo);
    if (g > sh->part_cap) {
      sh->part.alloc(sizeof(loopcore::Part) * g);
      sh->part_cap = g;
    }
    // fast path: slab x block layouts of the row and column slabs, indices
    // already in the gathered layout (x of a half = W blocks of stride doubles)
    const bool want_blk = !sh->log_domain && !ctx->deterministic && sh->m_own > 0 &&
                          (ctx->use_blocked == 1 || (ctx->use_blocked == 2 && n >= kBlockedAutoMinN));
    if (want_blk && !sh->blk_tried) {
      sh->blk_tried = true;
      if (!shard::blocked_shard_build(ctx, sh->m_own, (int64_t)sh->world * sh->stride, sh->rows.nnz, sh->rows.row_ptr,
                                      sh->rows.col_idx, sh->rows.values, sh->col_nnz, sh->col_ptr, sh->row_idx,
                                      sh->vals_t, (int)sh->vbytes, sh->blk))
        sh->blk.R.reset();
    }
    if (sh->blk.R && sh->blk.R->h.P > sh->part_cap) {
      sh->part.alloc(sizeof(loopcore::Part) * sh->blk.R->h.P);
      sh->part_cap = sh->blk.R->h.P;
    }
    shard::state_init_kernel<<<1, 1, 0, ctx->stream>>>(sh->state.as<shard::State>(), empty_rows_total,
                                                       empty_cols_total);
    shard::reset_kernel<<<1, 1, 0, ctx->stream>>>(sh->ticket.as<unsigned int>(), sh->flag.as<unsigned long long>());
    ctx->launches += 3;
    SPK_CUDA(cudaGetLastError());
    sh->calls = 0;
    sh->began = true;
  });
}

static int shard_step(spk_shard* sh, int half, int compute, int64_t t, const double* x_dev, const double* old_dev,
                      double* out_dev) {
  if (!sh) return SPK_STATUS_INPUT;
  return guard(sh->ctx, [&] {
    if (!sh->began) fail(SPK_E_LENGTH_MISMATCH, "call spk_shard_begin first");
    if (half != 0 && half != 1) fail(SPK_E_LENGTH_MISMATCH, "half must be 0 or 1");
    spk_ctx* ctx = sh->ctx;
    shard::HalfArgs A{};
    A.half = half;
    A.compute = compute && sh->m_own > 0;
    A.t = t;
    A.m_own = sh->m_own;
    A.base = sh->lo;
    A.m = sh->m;
    A.stride = sh->stride;
    A.world = sh->world;
    A.n = sh->n;
    A.max_iter = sh->max_iter;
    A.delta = sh->delta;
    A.exponent = sh->exponent;
    A.policy = sh->policy;
    const bool rows = half == 0;
    A.ptr = rows ? sh->rows.row_ptr.as<long long>() : sh->col_ptr.as<long long>();
    A.idx = rows ? sh->rows.col_idx.as<uint32_t>() : sh->row_idx.as<uint32_t>();
    A.val = rows ? sh->rows.values.p : sh->vals_t.p;
    A.x = x_dev;
    const int64_t own = (int64_t)sh->rank * sh->stride;
    A.old = old_dev ? old_dev + own : nullptr;
    A.out = out_dev ? out_dev + own : nullptr;
    A.w = sh->log_domain ? (rows ? sh->la : sh->lb).as<double>() : (rows ? sh->a : sh->b).as<double>();
    A.ne = (rows ? sh->row_ne : sh->col_ne).as<unsigned char>();
    A.dyn = (rows ? sh->dyn_row : sh->dyn_col).as<int>();
    shard::State* st = sh->state.as<shard::State>();
    A.st_in = st + (sh->calls & 1);
    A.st_out = st + ((sh->calls + 1) & 1);
    A.part = sh->part.as<loopcore::Part>();
    A.ticket = sh->ticket.as<unsigned int>();
    A.flag = sh->flag.as<unsigned long long>();
    const int grid = A.compute ? shard::grid_rows(ctx, sh->m_own) : 1;
    const bool f32 = sh->value_type == SPK_VALUES_F32;
    const bool blk = A.compute && !sh->log_domain && sh->blk.R && !ctx->deterministic &&
                     (ctx->use_blocked == 1 || (ctx->use_blocked == 2 && sh->n >= kBlockedAutoMinN));
    if (blk) {
      shard::blocked_shard_half(ctx, A, sh->blk);
      ++sh->calls;
      return;
    }
    if (sh->log_domain) {
      if (f32) launch_half<true, float>(sh, A, grid);
      else launch_half<true, double>(sh, A, grid);
    } else {
      if (f32) launch_half<false, float>(sh, A, grid);
      else launch_half<false, double>(sh, A, grid);
    }
    ++ctx->launches;
    ++sh->calls;
    SPK_CUDA(cudaGetLastError());
  });
}

int spk_shard_half(spk_shard* sh, int half, int64_t t, const double* x_dev, const double* old_dev, double* out_dev) {
  if (t < 1) return SPK_STATUS_INPUT;
  return shard_step(sh, half, 1, t, x_dev, old_dev, out_dev);
}

int spk_shard_finish(spk_shard* sh, int64_t t_last, const double* v_last_dev) {
  return shard_step(sh, 0, 0, t_last + 1, v_last_dev, nullptr, nullptr);
}

int spk_shard_status(spk_shard* sh, spk_report* rep, int32_t* stopped, int32_t* final_parity) {
  if (!sh) return SPK_STATUS_INPUT;
  return guard(sh->ctx, [&] {
    if (!sh->began) fail(SPK_E_LENGTH_MISMATCH, "call spk_shard_begin first");
    shard::State S;
    SPK_CUDA(cudaMemcpyAsync(&S, sh->state.as<shard::State>() + (sh->calls & 1), sizeof S, cudaMemcpyDeviceToHost,
                             sh->ctx->stream));
    SPK_CUDA(cudaStreamSynchronize(sh->ctx->stream));
    if (sh->blk.R) {  // slab x block halves record a barrier timeout instead of hanging
      unsigned int fw[2] = {0u, 0u};
      download(sh->ctx, fw, sh->blk.fault, sizeof fw);
      if (fw[0]) fail_device("sharded blocked half: a tile barrier timed out", cudaErrorLaunchTimeout);
    }
    if (stopped) *stopped = S.stopped;
    if (final_parity) *final_parity = S.final_par;
    if (rep) {
      rep->iterations = S.iterations;
      rep->converged = S.converged;
      rep->diverged = S.diverged;
      rep->masked_rows = S.masked_rows;
      rep->masked_cols = S.masked_cols;
      rep->log_domain = sh->log_domain;
      rep->kernel_nnz = sh->kernel_nnz;
      rep->factorized_plan = sh->factorized;
    }
    if (S.error_kind == SPK_E_ZERO_DENOMINATOR) {
      const std::string idx = std::to_string(S.error_index);
      if (sh->log_domain)
        fail(SPK_E_ZERO_DENOMINATOR, S.error_half == 0 ? "Kv vanished at row " + idx : "K'u vanished at column " + idx);
      fail(SPK_E_ZERO_DENOMINATOR, S.error_half == 0
                                       ? "Kv underflowed at row " + idx + "; consider SolverConfig::stabilize"
                                       : "K'u underflowed at column " + idx + "; consider SolverConfig::stabilize");
    }
    if (S.error_kind == SPK_E_DEGENERATE_SKETCH_ERROR) fail(SPK_E_DEGENERATE_SKETCH_ERROR, "masking removed every atom");
  });
}

int spk_shard_readout(spk_shard* sh, const double* u_dev, const double* v_dev, int log_domain, int uot,
                      int want_objective, double* out) {
  if (!sh || !out) return SPK_STATUS_INPUT;
  return guard(sh->ctx, [&] {
    spk_ctx* ctx = sh->ctx;
    if (!sh->imported) fail(SPK_E_LENGTH_MISMATCH, "column slab not imported yet");
    const int64_t mo = std::max<int64_t>(sh->m_own, 1);
    sh->rd_row_m.ensure(sizeof(double) * mo);
    sh->rd_col_m.ensure(sizeof(double) * mo);
    sh->rd_row_c.ensure(sizeof(double) * mo);
    sh->rd_row_h.ensure(sizeof(double) * mo);
    sh->rd_flags.ensure(3 * sizeof(unsigned long long));
    sh->rd_out.ensure(8 * sizeof(double));
    cudaStream_t s = ctx->stream;
    shard::fill3_kernel<<<1, 1, 0, s>>>(sh->rd_flags.as<unsigned long long>());
    SPK_CUDA(cudaMemsetAsync(sh->rd_out.p, 0, 8 * sizeof(double), s));
    const int64_t own = (int64_t)sh->rank * sh->stride;
    const CostSrc cs = cost_src_of(&sh->dk);
    const bool obj = want_objective != 0;
    unsigned long long* fl = sh->rd_flags.as<unsigned long long>();
    const int g = shard::grid_rows(ctx, mo);
#define SPK_READ(LOGV, VT)                                                                                           \
  do {                                                                                                               \
    if (obj)                                                                                                         \
      shard::read_rows_kernel<LOGV, true, VT><<<g, 512, 0, s>>>(                                                     \
          sh->m_own, sh->lo, sh->stride, sh->rows.row_ptr.as<long long>(), sh->rows.col_idx.as<uint32_t>(),          \
          sh->rows.values.as<VT>(), u_dev + own, v_dev, cs, sh->rd_row_m.as<double>(), sh->rd_row_c.as<double>(),    \
          sh->rd_row_h.as<double>(), fl);                                                                            \
    else                                                                                                             \
      shard::read_rows_kernel<LOGV, false, VT><<<g, 512, 0, s>>>(                                                    \
          sh->m_own, sh->lo, sh->stride, sh->rows.row_ptr.as<long long>(), sh->rows.col_idx.as<uint32_t>(),          \
          sh->rows.values.as<VT>(), u_dev + own, v_dev, cs, sh->rd_row_m.as<double>(), sh->rd_row_c.as<double>(),    \
          sh->rd_row_h.as<double>(), fl);                                                                            \
    shard::read_cols_kernel<LOGV, VT><<<g, 512, 0, s>>>(sh->m_own, sh->col_ptr.as<long long>(),                      \
                                                        sh->row_idx.as<uint32_t>(), sh->vals_t.as<VT>(), u_dev,      \
                                                        v_dev + own, sh->rd_col_m.as<double>());                     \
  } while (0)
    if (sh->m_own > 0) {
      const bool f32 = sh->value_type == SPK_VALUES_F32;
      if (log_domain) {
        if (f32) SPK_READ(true, float);
        else SPK_READ(true, double);
      } else {
        if (f32) SPK_READ(false, float);
        else SPK_READ(false, double);
      }
#undef SPK_READ
      shard::read_sums_kernel<<<1, 1024, 0, s>>>(sh->m_own, sh->lo, sh->rd_row_m.as<double>(),
                                                 sh->rd_col_m.as<double>(), sh->rd_row_c.as<double>(),
                                                 sh->rd_row_h.as<double>(), sh->a.as<double>(), sh->b.as<double>(),
                                                 obj ? 1 : 0, uot, fl + 1, sh->rd_out.as<double>());
      ctx->launches += 3;
    }
    double sums[8];
    unsigned long long flags[3];
    download(ctx, sums, sh->rd_out, sizeof(double) * 6);
    download(ctx, flags, sh->rd_flags, sizeof flags);
    for (int k = 0; k < 6; ++k) out[k] = sums[k];
    out[6] = flags[0] == shard::kNone ? 0.0 : (double)flags[0] + 1.0;
    const unsigned long long kb = std::min(flags[1], flags[2]);
    out[7] = kb == shard::kNone ? 0.0 : (double)kb + 1.0;
    SPK_CUDA(cudaGetLastError());
  });
}

}  // extern "C"
