// rowdot.cuh -- one warp's dot product of a sparse row (CSR row or CSC column)
// with a gathered scaling vector, linear or log-sum-exp; shared by the
// single-GPU loop (loop.cu) and the sharded half-steps (shard.cu).
#pragma once

#include "common.cuh"

namespace spk {

// A sketch value that already holds log K~ (the log-domain loop precomputes
// them once per sketch instead of taking a log per entry per iteration).
struct LogK {
  double v;
};
__device__ __forceinline__ double log_of(double v) { return log(v); }
__device__ __forceinline__ double log_of(float v) { return log((double)v); }
__device__ __forceinline__ double log_of(LogK v) { return v.v; }
__device__ __forceinline__ double ldg_val(const double* p) { return __ldg(p); }
__device__ __forceinline__ float ldg_val(const float* p) { return __ldg(p); }
__device__ __forceinline__ LogK ldg_val(const LogK* p) { return LogK{__ldg(&p->v)}; }

// Row value of one half: sum_p val[p] * x[idx[p]] over [b, e) (linear), or
// the log-sum-exp of log(val[p]) + x[idx[p]] skipping x = -inf (log).
template <bool LOG, bool DET, class VT>
__device__ __forceinline__ double row_apply(const VT* __restrict__ val, const uint32_t* __restrict__ idx, long long b,
                                            long long e, const double* x, int lane) {
  if constexpr (!LOG) {
    if (DET) {  // acc += v * x, j ascending, no FMA (sparsify.cpp:208-209)
      double acc = 0.0;
      for (long long p = b; p < e; ++p) acc = dadd(acc, dmul((double)val[p], __ldcg(x + idx[p])));
      return acc;
    }
    double a0 = 0.0, a1 = 0.0;
    long long p = b + lane;
    for (; p + 32 < e; p += 64) {
      const uint32_t c0 = __ldg(idx + p), c1 = __ldg(idx + p + 32);
      const double w0 = (double)__ldg(val + p), w1 = (double)__ldg(val + p + 32);
      a0 = fma(w0, __ldcg(x + c0), a0);
      a1 = fma(w1, __ldcg(x + c1), a1);
    }
    if (p < e) a0 = fma((double)__ldg(val + p), __ldcg(x + __ldg(idx + p)), a0);
    return warp_sum(a0 + a1);
  } else {
    if (DET) {  // two passes: max, then the shifted sum (solvers.cpp:99-111)
      double mx = -CUDART_INF;
      for (long long p = b; p < e; ++p) {
        const double xv = __ldcg(x + idx[p]);
        if (xv == -CUDART_INF) continue;
        mx = fmax(mx, dadd(log_of(val[p]), xv));
      }
      if (mx == -CUDART_INF) return -CUDART_INF;
      double acc = 0.0;
      for (long long p = b; p < e; ++p) {
        const double xv = __ldcg(x + idx[p]);
        if (xv == -CUDART_INF) continue;
        acc = dadd(acc, exp(dsub(dadd(log_of(val[p]), xv), mx)));
      }
      return dadd(mx, log(acc));
    }
    // online (max, scaled sum) per lane, merged across the warp
    double m = -CUDART_INF, s = 0.0;
    for (long long p = b + lane; p < e; p += 32) {
      const double xv = __ldcg(x + __ldg(idx + p));
      if (xv == -CUDART_INF) continue;
      const double t = log_of(ldg_val(val + p)) + xv;
      if (t == -CUDART_INF) continue;  // a zero K~ (e.g. fp32 underflow) adds nothing
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
}

}  // namespace spk
