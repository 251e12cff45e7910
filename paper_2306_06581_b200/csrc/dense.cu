// dense.cu -- dense Sinkhorn half-step operators (north-star item 5)
// for the persistent loop in loop_core.cuh.
//
// Reference: sinkhorn_ot / sinkhorn_uot on a KernelMatrix (include/sparsink/solvers.hpp:137-147)
// with kernel_apply / kernel_apply_t (proj/src/solvers.cpp:12-34) and
// kernel_log_apply(_t) (:52-94); default EmptyPolicy::Error.
//
// Three operators:
//   DenseOp     K uploaded (n x n fp64): rows as warp dot products; columns one
//               thread per column walking rows in order -- coalesced AND the
//               reference's kernel_apply_t summation order.
//   OtfExactOp  K_ij = exp(-C_ij/eps) recomputed in fp64 from coordinates
//               every iteration (exact kernel_from_cost values, no n^2 memory).
//   OtfFastOp   config-5 comparator: squared-Euclidean K recomputed every
//               iteration in fp32 as exp2(A_i + B_j + <x'_i, y_j>) (one MUFU.EX2
//               + 6 FFMA per entry), fp32 partial sums per 256-column chunk
//               folded into fp64. SFU/FMA-bound, no n^2 memory.
#include <algorithm>
#include <cmath>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "ksrc.cuh"
#include "loop_core.cuh"

#include <cooperative_groups.h>

namespace spk {

namespace {

using loopcore::finalize_atom;

// Shared body for dense/exact operators: ROLE 0 = rows, ROLE 1 = columns.
template <class KF>
struct ExactOp {
  static constexpr int kThreads = loopcore::kBlock;
  static constexpr int kMinBlocks = 2;
  KF k;
  int64_t n;

  template <bool LOG, bool DET>
  __device__ double row_value(int64_t i, const double* x, int lane) const {
    if (!LOG) {
      if (DET) {
        double acc = 0.0;
        for (int64_t j = 0; j < n; ++j) acc = dadd(acc, dmul(k(i, j), __ldcg(x + j)));
        return acc;
      }
      double acc = 0.0;
      for (int64_t j = lane; j < n; j += 32) acc = fma(k(i, j), __ldcg(x + j), acc);
      return warp_sum(acc);
    }
    // kernel_log_apply dense (solvers.cpp:52-71)
    if (DET) {
      double mx = -CUDART_INF;
      for (int64_t j = 0; j < n; ++j) {
        const double kij = k(i, j), xv = __ldcg(x + j);
        if (kij == 0.0 || xv == -CUDART_INF) continue;
        mx = fmax(mx, dadd(log(kij), xv));
      }
      if (mx == -CUDART_INF) return -CUDART_INF;
      double acc = 0.0;
      for (int64_t j = 0; j < n; ++j) {
        const double kij = k(i, j), xv = __ldcg(x + j);
        if (kij == 0.0 || xv == -CUDART_INF) continue;
        acc = dadd(acc, exp(dsub(dadd(log(kij), xv), mx)));
      }
      return dadd(mx, log(acc));
    }
    double m = -CUDART_INF, s = 0.0;
    for (int64_t j = lane; j < n; j += 32) {
      const double kij = k(i, j), xv = __ldcg(x + j);
      if (kij == 0.0 || xv == -CUDART_INF) continue;
      const double t = log(kij) + xv;
      if (t > m) {
        s = s * exp(m - t) + 1.0;
        m = t;
      } else {
        s += exp(t - m);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const double s2 = __shfl_xor_sync(0xffffffffu, s, o);
      const double M = fmax(m, m2);
      if (M != -CUDART_INF)
        s = (m == -CUDART_INF ? 0.0 : s * exp(m - M)) + (m2 == -CUDART_INF ? 0.0 : s2 * exp(m2 - M));
      m = M;
    }
    return m == -CUDART_INF ? -CUDART_INF : m + log(s);
  }

  // Column j: rows in ascending order, skipping u_i == 0 (solvers.cpp:28-33)
  // or lu_i = -inf (:77-93). One thread per column.
  template <bool LOG>
  __device__ double col_value(int64_t j, const double* x) const {
    if (!LOG) {
      double acc = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        const double xi = __ldcg(x + i);
        if (xi == 0.0) continue;
        acc = dadd(acc, dmul(k(i, j), xi));
      }
      return acc;
    }
    double mx = -CUDART_INF;
    for (int64_t i = 0; i < n; ++i) {
      const double xi = __ldcg(x + i);
      const double kij = k(i, j);
      if (xi == -CUDART_INF || !(kij > 0.0)) continue;
      mx = fmax(mx, dadd(log(kij), xi));
    }
    if (mx == -CUDART_INF) return -CUDART_INF;
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double xi = __ldcg(x + i);
      const double kij = k(i, j);
      if (xi == -CUDART_INF || !(kij > 0.0)) continue;
      acc = dadd(acc, exp(dsub(dadd(log(kij), xi), mx)));
    }
    return dadd(mx, log(acc));
  }

  template <int ROLE, bool LOG, bool DET>
  __device__ void half(const double* x, const double* wgt, const double* old, double* out, unsigned char* ne,
                       int* dyn, double exponent, int policy, int t, unsigned long long* flag, double* absdiff,
                       double& err, long long& masks) const {
    const int lane = threadIdx.x & 31;
    if (ROLE == 1 || DET) {
      const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
      const int64_t nth = (int64_t)gridDim.x * blockDim.x;
      for (int64_t i = tid; i < n; i += nth) {
        double d = 0.0;
        const double o = __ldcg(old + i);
        if (ne[i]) {
          const double tmp = ROLE == 0 ? row_value<LOG, true>(i, x, lane) : col_value<LOG>(i, x);
          d = finalize_atom<LOG>(i, tmp, o, wgt[i], exponent, policy, t, ne, dyn, out, flag, masks);
        } else {
          out[i] = o;
        }
        if (DET) absdiff[i] = d;
        else err += d;
      }
    } else {
      const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
      const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
      for (int64_t i = warp; i < n; i += nw) {
        if (!ne[i]) {
          if (lane == 0) out[i] = __ldcg(old + i);
          continue;
        }
        const double tmp = row_value<LOG, false>(i, x, lane);
        if (lane == 0) err += finalize_atom<LOG>(i, tmp, __ldcg(old + i), wgt[i], exponent, policy, t, ne, dyn, out, flag, masks);
      }
    }
  }
};

// ---- fast fp32 on-the-fly squared-Euclidean operator (config 5) ---------------

constexpr int kOtfDim = 8;     // padded point record: d <= 6 coords + bias
constexpr int kOtfRows = 4;    // rows per lane
constexpr int kOtfChunk = 256; // columns per fp32 partial

// Point records (float4 x2): {p_0..p_{d-1}, bias, 0...}. For the output side
// p = -2*alpha*x_i and bias = alpha*|x_i|^2; input side p = y_j, bias =
// alpha*|y_j|^2, with alpha = -log2(e)/(scale*eps), so
// K_ij = exp2(bias_i + bias_j + <p_i, y_j>) = exp(-|x_i - y_j|^2/(scale*eps)).
// MUFU.EX2 with subnormal results flushed to zero: K values below 2^-126
// (the fp32 comparator's own floor is 2^-149) count as zero. Saves the
// range test and two multiplies exp2f spends per kernel evaluation.
__device__ __forceinline__ float ex2_ftz(float e) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e));
  return r;
}

// FOLD: the input side's bias_j = alpha |y_j|^2 is folded into its scaling
// (x'_j = x_j exp2(bias_j), once per half) so an evaluation is exp2(bias_i +
// <p_i, y_j>) * x'_j: D FMA-pipe ops for the exponent instead of D + 1. Used
// only when |alpha| max |pt|^2 <= 60, so neither exp2(bias_i + <p_i, y_j>) =
// exp2(e_ij - bias_j) can overflow nor exp2(bias_j) underflow.
template <int D, bool FOLD>
struct OtfFastOp {
  static constexpr int kThreads = loopcore::kBlock;
  static constexpr int kMinBlocks = 1;  // 128 registers (at 64 the point records spill)
  int64_t n;
  int dim;
  const float4* out_rec[2];  // [role] output-side records (2 float4 per atom)
  const float4* in_rec[2];   // [role] input-side records
  int parts;                 // column ranges per row block (work items ~ warps of the grid)
  double* partial;           // [parts][n] partial row sums
  float* xf;                 // [n + 4] fp32 copy of the gathered scalings of the half
  const float* colscale[2];  // [role] FOLD: exp2(bias_j) of the input side

  // exponent of K_ij in log2 units: bias_i + bias_j + <p_i, y_j>, D + 1 FMA-pipe ops
  __device__ __forceinline__ static float expo(const float (&p)[D + 1], const float (&q)[8]) {
    float e = FOLD ? p[D] : p[D] + q[7];
#pragma unroll
    for (int k = 0; k < D; ++k) e = fmaf(p[k], q[k], e);
    return e;
  }
  __device__ __forceinline__ static void load_rec(const float4* rp, float (&q)[8]) {
    const float4 a = __ldg(rp);
    q[0] = a.x; q[1] = a.y; q[2] = a.z; q[3] = a.w;
    if (D > 3) {  // d <= 3: coordinates + bias fit the first float4... the bias lives in slot 7
      const float4 b = __ldg(rp + 1);
      q[4] = b.x; q[5] = b.y; q[6] = b.z; q[7] = b.w;
    } else {
      const float4 b = __ldg(rp + 1);
      q[7] = b.w;
    }
  }

  // Work item = (a group of 16 row blocks of 32 x kOtfRows rows, one per
  // warp) x (one of `parts` column ranges), one CTA each. The CTA streams the
  // range's column records and scalings through shared memory in chunks of
  // kOtfChunk columns (cp.async, double-buffered): every warp reads them as
  // broadcast LDS instead of each warp fetching them from L2. Items go to
  // CTAs round-robin (items ~ a multiple of the grid). Each warp leaves fp64
  // partial row sums in partial[cp * n + i]; after one grid barrier the rows
  // are finalised from their `parts` partials summed in column-range order.
  static constexpr int kWarps = loopcore::kBlock / 32;
  static constexpr int kChunkRecBytes = kOtfChunk * 32;  // 2 float4 per column
  static constexpr int kChunkXBytes = kOtfChunk * 4;  // fp32 copy of the scalings
  static constexpr int kStageBytes = kChunkRecBytes + kChunkXBytes;

  __device__ static void stage_chunk(char* dst, const float4* irec, const float* x, int64_t c0, int len) {
    // records: len * 32 bytes, x: len * 4 bytes (16-byte cp.async pieces; tails zero-filled)
    const char* rs = reinterpret_cast<const char*>(irec + 2 * c0);
    for (int k = threadIdx.x; k < kChunkRecBytes / 16; k += blockDim.x) {
      const int col = k >> 1;
      void* d = dst + 16 * k;
      if (col < len) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(d)),
                     "l"(rs + 16 * k)
                     : "memory");
      } else {
        *reinterpret_cast<float4*>(d) = make_float4(0.f, 0.f, 0.f, 0.f);  // finite exp2, times x = 0 below
      }
    }
    const char* xs = reinterpret_cast<const char*>(x + c0);
    for (int k = threadIdx.x; k < kChunkXBytes / 16; k += blockDim.x) {
      void* d = dst + kChunkRecBytes + 16 * k;
      if (4 * k + 3 < len) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(d)),
                     "l"(xs + 16 * k)
                     : "memory");
      } else {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (4 * k < len) v.x = __ldcg(x + c0 + 4 * k);
        if (4 * k + 1 < len) v.y = __ldcg(x + c0 + 4 * k + 1);
        if (4 * k + 2 < len) v.z = __ldcg(x + c0 + 4 * k + 2);
        *reinterpret_cast<float4*>(d) = v;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }

  template <int ROLE, bool LOG, bool DET>
  __device__ void half(const double* x, const double* wgt, const double* old, double* out, unsigned char* ne,
                       int* dyn, double exponent, int policy, int t, unsigned long long* flag, double* absdiff,
                       double& err, long long& masks) const {
    __shared__ __align__(16) char stage[2][kStageBytes];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const float4* orec = out_rec[ROLE];
    const float4* irec = in_rec[ROLE];
    // fp32 copy of the gathered scalings, once per half (one conversion per
    // column instead of one per column per warp: the conversions share the
    // MUFU pipe with the exp2s)
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
      xf[j] = FOLD ? (float)__ldcg(x + j) * __ldg(colscale[ROLE] + j) : (float)__ldcg(x + j);
    cooperative_groups::this_grid().sync();
    const int64_t tile_rows = 32 * kOtfRows;
    const int64_t nrb = (n + tile_rows - 1) / tile_rows;
    const int64_t ngroups = (nrb + kWarps - 1) / kWarps;
    const int64_t items = ngroups * parts;
    const int64_t per = ((n + parts - 1) / parts + 3) & ~int64_t(3);  // columns per range (multiple of 4: 16-byte fp32 x pieces)
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
      const int64_t grp = item / parts;
      const int cp = (int)(item - grp * parts);
      const int64_t rbk = grp * kWarps + w;  // this warp's row block
      const int64_t r0 = rbk * tile_rows;
      const int64_t c_lo = min(n, cp * per), c_hi = min(n, c_lo + per);
      float p[kOtfRows][D + 1];
      double acc[kOtfRows];
#pragma unroll
      for (int r = 0; r < kOtfRows; ++r) {
        const int64_t i = r0 + lane + 32 * r;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        if (i < n) {
          a = orec[2 * i];
          b = orec[2 * i + 1];
        }
        const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < D; ++k) p[r][k] = v[k];
        p[r][D] = v[7];  // bias_i
        acc[r] = 0.0;
      }
      const int nch = (int)((c_hi - c_lo + kOtfChunk - 1) / kOtfChunk);
      __syncthreads();  // the previous item's readers of the stage buffers are done
      if (nch > 0) stage_chunk(stage[0], irec, xf, c_lo, (int)min((int64_t)kOtfChunk, c_hi - c_lo));
      for (int ch = 0; ch < nch; ++ch) {
        const int64_t c0 = c_lo + (int64_t)ch * kOtfChunk;
        const int len = (int)min((int64_t)kOtfChunk, c_hi - c0);
        if (ch + 1 < nch) {  // next chunk in flight while this one computes
          const int64_t c1 = c0 + kOtfChunk;
          stage_chunk(stage[(ch + 1) & 1], irec, xf, c1, (int)min((int64_t)kOtfChunk, c_hi - c1));
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();  // chunk ch staged by every thread
        const float4* qs = reinterpret_cast<const float4*>(stage[ch & 1]);
        const float* xs = reinterpret_cast<const float*>(stage[ch & 1] + kChunkRecBytes);
        float part[kOtfRows];
#pragma unroll
        for (int r = 0; r < kOtfRows; ++r) part[r] = 0.f;
        if (r0 < n) {
          for (int jj = 0; jj < len; jj += 2) {  // two columns per step (a zero-filled odd tail adds 0)
            float q0[8], q1[8];
            {
              const float4 a0 = qs[2 * jj], b0 = qs[2 * jj + 1], a1 = qs[2 * jj + 2], b1 = qs[2 * jj + 3];
              q0[0] = a0.x; q0[1] = a0.y; q0[2] = a0.z; q0[3] = a0.w;
              q0[4] = b0.x; q0[5] = b0.y; q0[6] = b0.z; q0[7] = b0.w;
              q1[0] = a1.x; q1[1] = a1.y; q1[2] = a1.z; q1[3] = a1.w;
              q1[4] = b1.x; q1[5] = b1.y; q1[6] = b1.z; q1[7] = b1.w;
            }
            const float2 xd = *reinterpret_cast<const float2*>(xs + jj);
            const float x0 = xd.x, x1 = xd.y;
#pragma unroll
            for (int r = 0; r < kOtfRows; ++r) {
              const float e0 = expo(p[r], q0), e1 = expo(p[r], q1);
              part[r] = fmaf(ex2_ftz(e0), x0, part[r]);
              part[r] = fmaf(ex2_ftz(e1), x1, part[r]);
            }
          }
        }
#pragma unroll
        for (int r = 0; r < kOtfRows; ++r) acc[r] += (double)part[r];
        __syncthreads();  // every warp is done with chunk ch before its buffer is refilled
      }
#pragma unroll
      for (int r = 0; r < kOtfRows; ++r) {
        const int64_t i = r0 + lane + 32 * r;
        if (i < n) partial[(int64_t)cp * n + i] = acc[r];
      }
    }
    cooperative_groups::this_grid().sync();  // every partial row sum written
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      double tmp = 0.0;
      for (int c = 0; c < parts; ++c) tmp += __ldcg(partial + (int64_t)c * n + i);  // column-range order
      const double o = __ldcg(old + i);
      if (!ne[i]) {
        out[i] = o;
        continue;
      }
      err += finalize_atom<false>(i, tmp, o, wgt[i], exponent, policy, t, ne, dyn, out, flag, masks);
    }
  }
};

// Coverage of a dense / on-the-fly kernel: row i covered iff some K_ij > 0
// (solvers.cpp:138-152).
template <class KF>
__global__ void dense_coverage_kernel(KF k, int64_t n, unsigned char* row_ne, unsigned char* col_ne,
                                      unsigned long long* empty) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < 2 * n; i += nw) {
    const bool rowside = i < n;
    const int64_t a = rowside ? i : i - n;
    bool any = false;
    for (int64_t j = lane; j < n && !any; j += 32) any = (rowside ? k(a, j) : k(j, a)) > 0.0;
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) {
      (rowside ? row_ne : col_ne)[a] = any ? 1 : 0;
      if (!any) atomicAdd(&empty[rowside ? 0 : 1], 1ull);
    }
  }
}

template <bool LOG, class KF>
void run_exact(spk_ctx* ctx, KF kf, int64_t n, const spk_solver_cfg& cfg, double exponent, int policy,
               LoopState& st, LoopOut& out) {
  LoopWs W;
  W.row_ne.alloc(n);
  W.col_ne.alloc(n);
  DBuf empty(16);
  SPK_CUDA(cudaMemsetAsync(empty.p, 0, 16, ctx->stream));
  dense_coverage_kernel<KF><<<(int)std::max<int64_t>(1, std::min<int64_t>((2 * n + 7) / 8, ctx->num_sms * 16)), 256, 0,
                              ctx->stream>>>(kf, n, W.row_ne.as<unsigned char>(), W.col_ne.as<unsigned char>(),
                                             empty.as<unsigned long long>());
  ++ctx->launches;
  unsigned long long emp[2];
  download(ctx, emp, empty, sizeof emp);
  ExactOp<KF> op;
  op.k = kf;
  op.n = n;
  const int64_t useful = (n + 15) / 16;
  loopcore::run_core<LOG>(ctx, op, n, W, (long long)emp[0], (long long)emp[1], cfg, exponent, policy, st, useful,
                          out);
}

__global__ void otf_records_kernel(const double* pts, int64_t n, int dim, double alpha, float4* out_rec,
                                   float4* in_rec, float* in_scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float o[kOtfDim] = {0, 0, 0, 0, 0, 0, 0, 0};
    float q[kOtfDim] = {0, 0, 0, 0, 0, 0, 0, 0};
    double nrm = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double c = pts[i * dim + k];
      nrm += c * c;
      o[k] = (float)(-2.0 * alpha * c);
      q[k] = (float)c;
    }
    o[7] = (float)(alpha * nrm);
    q[7] = (float)(alpha * nrm);
    out_rec[2 * i] = make_float4(o[0], o[1], o[2], o[3]);
    out_rec[2 * i + 1] = make_float4(o[4], o[5], o[6], o[7]);
    in_rec[2 * i] = make_float4(q[0], q[1], q[2], q[3]);
    in_rec[2 * i + 1] = make_float4(q[4], q[5], q[6], q[7]);
    in_scale[i] = exp2f((float)(alpha * nrm));  // FOLD: exp2(bias) of this point as an input
  }
}

}  // namespace

void run_dense_loop(spk_ctx* ctx, DevKernel& dk, const spk_solver_cfg& cfg, double exponent, int policy,
                    LoopState& st, LoopOut& out) {
  const int64_t n = dk.n;
  const bool log_domain = cfg.stabilize != 0;
  if (dk.dense) {
    KDense kf{dk.K.as<double>(), n};
    if (log_domain) run_exact<true>(ctx, kf, n, cfg, exponent, policy, st, out);
    else run_exact<false>(ctx, kf, n, cfg, exponent, policy, st, out);
    return;
  }
  const bool fast = !ctx->deterministic && !log_domain && ctx->otf_fp32 && dk.kind == SPK_COST_SQEUCLID && dk.dim <= 6;
  if (!fast) {
    KCoords kf = kcoords_of(dk);
    if (log_domain) run_exact<true>(ctx, kf, n, cfg, exponent, policy, st, out);
    else run_exact<false>(ctx, kf, n, cfg, exponent, policy, st, out);
    return;
  }
  // fp32 records for both roles
  DBuf xo(sizeof(float4) * 2 * n), xi(sizeof(float4) * 2 * n), yo(sizeof(float4) * 2 * n), yi(sizeof(float4) * 2 * n);
  const double alpha = -1.4426950408889634 / (dk.scale * dk.eps);
  const int g = loopcore::simple_grid(ctx, n);
  DBuf xs(sizeof(float) * n), ys(sizeof(float) * n);
  otf_records_kernel<<<g, 256, 0, ctx->stream>>>(dk.x.as<double>(), n, dk.dim, alpha, xo.as<float4>(), xi.as<float4>(),
                                                 xs.as<float>());
  otf_records_kernel<<<g, 256, 0, ctx->stream>>>(dk.y.as<double>(), n, dk.dim, alpha, yo.as<float4>(), yi.as<float4>(),
                                                 ys.as<float>());
  // fold the input bias into the scalings when no exp2 can leave the fp32 range
  const bool fold = std::fabs(alpha) * dk.dim * dk.max_abs * dk.max_abs <= 60.0;
  ctx->launches += 2;
  const float4* recs[4] = {xo.as<float4>(), yi.as<float4>(), yo.as<float4>(), xi.as<float4>()};
  // coverage: exp2 of finite exponents never reaches 0 for max-normalised
  // costs with 1/eps < 700; otherwise use the exact coverage pass.
  LoopWs W;
  W.row_ne.alloc(n);
  W.col_ne.alloc(n);
  DBuf empty(16);
  SPK_CUDA(cudaMemsetAsync(empty.p, 0, 16, ctx->stream));
  KCoords kf = kcoords_of(dk);
  dense_coverage_kernel<KCoords><<<(int)std::max<int64_t>(1, std::min<int64_t>((2 * n + 7) / 8, ctx->num_sms * 16)),
                                   256, 0, ctx->stream>>>(kf, n, W.row_ne.as<unsigned char>(),
                                                          W.col_ne.as<unsigned char>(), empty.as<unsigned long long>());
  ++ctx->launches;
  unsigned long long emp[2];
  download(ctx, emp, empty, sizeof emp);
  // grid = co-resident CTAs (run_core: occupancy x SMs); pick the column
  // ranges so that (row blocks x ranges) matches the grid's warps
  int per_sm = 1;
  {
    auto k5 = loopcore::loop_kernel<false, false, OtfFastOp<5, true>>;  // (all variants share the occupancy)
    SPK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k5, loopcore::kBlock, 0));
    per_sm = std::max(per_sm, 1);
  }
  // CTA items = (groups of 16 row blocks) x parts: a whole number of rounds
  // over the co-resident CTAs, >= 4 rounds so a short last group costs little
  const int64_t nrb = (n + 32 * kOtfRows - 1) / (32 * kOtfRows);
  const int64_t ngroups = (nrb + loopcore::kBlock / 32 - 1) / (loopcore::kBlock / 32);
  const int64_t ctas = (int64_t)ctx->num_sms * per_sm;
  int parts = 1;
  {
    double best = 0.0;
    for (int pp = 1; pp <= 128; ++pp) {
      const int64_t items = ngroups * pp;
      const int64_t rounds = (items + ctas - 1) / ctas;
      const int64_t cols = (n + pp - 1) / pp;
      if (cols < 2 * kOtfChunk && pp > 1) break;  // ranges shorter than two chunks: staging overhead
      const double eff = (double)items / (double)(rounds * ctas);
      if (eff > best + 1e-9) {
        best = eff;
        parts = pp;
      }
      if (eff > 0.97 && rounds >= 2) break;
    }
  }
  DBuf partial(sizeof(double) * (size_t)parts * n);
  DBuf xf(sizeof(float) * ((size_t)n + 4));
  const int64_t useful = (int64_t)ctx->num_sms * per_sm;
  // the point-record width is a compile-time constant: D + 1 FMA-pipe ops per evaluation
  auto go2 = [&](auto dtag, auto ftag) {
    constexpr int D = decltype(dtag)::value;
    constexpr bool FOLD = decltype(ftag)::value;
    OtfFastOp<D, FOLD> op;
    op.colscale[0] = ys.as<float>();  // rows: inputs are the y points
    op.colscale[1] = xs.as<float>();
    op.n = n;
    op.dim = dk.dim;
    op.out_rec[0] = recs[0];  // rows: x_i against y_j
    op.in_rec[0] = recs[1];
    op.out_rec[1] = recs[2];  // columns: y_j against x_i
    op.in_rec[1] = recs[3];
    op.parts = parts;
    op.partial = partial.as<double>();
    op.xf = xf.as<float>();
    loopcore::run_core<false>(ctx, op, n, W, (long long)emp[0], (long long)emp[1], cfg, exponent, policy, st,
                              useful, out);
  };
  auto go = [&](auto dtag) {
    if (fold) go2(dtag, std::true_type{});
    else go2(dtag, std::false_type{});
  };
  switch (dk.dim) {
    case 1: go(std::integral_constant<int, 1>{}); break;
    case 2: go(std::integral_constant<int, 2>{}); break;
    case 3: go(std::integral_constant<int, 3>{}); break;
    case 4: go(std::integral_constant<int, 4>{}); break;
    case 5: go(std::integral_constant<int, 5>{}); break;
    default: go(std::integral_constant<int, 6>{}); break;
  }
}

}  // namespace spk
