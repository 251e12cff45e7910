// rowdot.cuh -- one warp's dot product of a sparse row (CSR row or CSC column)
// with a gathered scaling vector, linear or log-sum-exp; shared by the
// single-GPU loop (loop.cu) and the sharded half-steps (shard.cu).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace spk {

// A sketch value that already holds log K~ (the log-domain loop precomputes
// them once per sketch instead of taking a log per entry per iteration).
struct LogK {
  double v;
};
// The same, for a sketch stored in fp32: its log-sum-exp terms take an
// fp32-accurate exp (MUFU.EX2, relative error ~2^-22, the order of the fp32
// rounding of K~ itself; sums and logs stay fp64).
struct LogKf {
  double v;
};
__device__ __forceinline__ double log_of(double v) { return log(v); }
__device__ __forceinline__ double log_of(float v) { return log((double)v); }
__device__ __forceinline__ double log_of(LogK v) { return v.v; }
__device__ __forceinline__ double log_of(LogKf v) { return v.v; }
__device__ __forceinline__ LogKf ldg_val(const LogKf* p) { return LogKf{__ldg(&p->v)}; }

// exp(d) for d <= 0 (a log-sum-exp term): fp64, or fp32-accurate for fp32 sketches
__device__ __forceinline__ double exp_fast(double d) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)(d * 1.4426950408889634)));
  return (double)r;
}
template <class VT>
__device__ __forceinline__ double exp_term(double d) {
  if constexpr (std::is_same<VT, LogKf>::value) return exp_fast(d);
  else return exp(d);
}
__device__ __forceinline__ double ldg_val(const double* p) { return __ldg(p); }
__device__ __forceinline__ float ldg_val(const float* p) { return __ldg(p); }
__device__ __forceinline__ LogK ldg_val(const LogK* p) { return LogK{__ldg(&p->v)}; }

// Row value of one half: sum_p val[p] * x[idx[p]] over [b, e) (linear), or
// the log-sum-exp of log(val[p]) + x[idx[p]] skipping x = -inf (log).
// XS: x is a copy staged in shared memory (plain loads); else the global
// vector, read through L2 (it is rewritten inside the same launch).
template <bool XS>
__device__ __forceinline__ double ld_x(const double* x, uint32_t c) {
  if constexpr (XS) return x[c];
  else return __ldcg(x + c);
}

template <bool LOG, bool DET, class VT, bool XS = false>
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
      a0 = fma(w0, ld_x<XS>(x, c0), a0);
      a1 = fma(w1, ld_x<XS>(x, c1), a1);
    }
    if (p < e) a0 = fma((double)__ldg(val + p), ld_x<XS>(x, __ldg(idx + p)), a0);
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
    // two passes (the reference's order of operations, solvers.cpp:99-111):
    // the row max (no exp), then the sum of exp(t - max) -- one exp per
    // entry; the warp merges are a plain max and a plain sum
    double m = -CUDART_INF;
    for (long long p = b + lane; p < e; p += 32) {
      const double xv = ld_x<XS>(x, __ldg(idx + p));
      if (xv == -CUDART_INF) continue;
      m = fmax(m, log_of(ldg_val(val + p)) + xv);
    }
    m = warp_max(m);
    if (m == -CUDART_INF) return -CUDART_INF;
    double s = 0.0;
    for (long long p = b + lane; p < e; p += 32) {
      const double xv = ld_x<XS>(x, __ldg(idx + p));
      if (xv == -CUDART_INF) continue;
      s += exp_term<VT>(log_of(ldg_val(val + p)) + xv - m);  // a zero K~ (log -inf) adds exp(-inf) = 0
    }
    return m + log(warp_sum(s));
  }
}

}  // namespace spk
