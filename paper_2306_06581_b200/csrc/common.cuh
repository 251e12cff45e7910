// common.cuh -- device helpers shared by the Spar-Sink kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

namespace spk {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
constexpr int kWarp = 32;

// splitmix64 finalizer without the increment: the t-th draw of the
// reference's CounterRng(seed, stream) is finalize(mix_seed(seed,stream) +
// t*golden) (rng.hpp:29-35). Integer pipe only.
__host__ __device__ __forceinline__ uint64_t sm_finalize(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {  // rng.hpp:10-15
  return sm_finalize(x + kGolden);
}
__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t seed, uint64_t stream) {  // rng.hpp:17-19
  return splitmix64(seed ^ splitmix64(stream + 0x632be59bd9b4e019ULL));
}
// next_double (rng.hpp:38-40): top 53 bits scaled by 2^-53 (exact).
__device__ __forceinline__ double u64_to_unit(uint64_t x) {
  return __dmul_rn(__ull2double_rn(x >> 11), 0x1.0p-53);
}

// Exact (contraction-free) arithmetic for reference-order sums.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// pairwise_cost entry (geometry.cpp:16-59) in the reference's operation
// order with no FMA: sequential d2, then the per-kind transform.
template <int KIND>
__device__ __forceinline__ double cost_from_d2(double d2, double eta) {
  if (KIND == 0) return d2;
  if (KIND == 1) return sqrt(d2);
  const double d = sqrt(d2);
  if (d >= dmul(3.14159265358979323846, eta)) return CUDART_INF;
  const double cz = cos(d / dmul(2.0, eta));
  double v = -log(dmul(cz, cz));
  if (!(v >= 0.0)) v = 0.0;
  return v;
}

__device__ __forceinline__ double cost_from_d2_rt(int kind, double d2, double eta) {
  if (kind == 0) return cost_from_d2<0>(d2, eta);
  if (kind == 1) return cost_from_d2<1>(d2, eta);
  return cost_from_d2<2>(d2, eta);
}

// exp(x) with the reference's (glibc's) underflow boundary. K != 0 decides
// the sketch support and therefore every later draw counter of the row
// (sparsify.cpp:184-198), so the boundary must be bit-exact: glibc's exp is
// correctly rounded there -- exp(x) != 0 exactly for x >= -0x1.74910d52d3051p+9,
// the double just above -1075 ln 2 (tests/test_exp_boundary.py re-derives it
// from the host libm) -- while CUDA's exp flushes part of the deepest subnormal
// range to 0 (config 4: 142 of 10^12 pairs). Subnormal results are formed as
// rint(e^(x + 1074 ln 2)) quanta of 2^-1074 (Cody-Waite split of 1074 ln 2; the
// first sum is exact by Sterbenz), within a few quanta of glibc's value.
constexpr double kExpLastNonzero = -0x1.74910d52d3051p+9;  // glibc: exp(x) == 2^-1074 here, 0 below
constexpr double kExpSubnormal = -708.39641853226408;      // ln(2^-1022): below, results are subnormal
__device__ __forceinline__ double exp_ref(double x) {
  if (!(x < kExpSubnormal)) return exp(x);  // normal results (and NaN, +-inf handled by exp)
  if (x < kExpLastNonzero) return 0.0;
  constexpr double kHi = 1074.0 * 0x1.62e42feep-1;  // ln2_hi (21 trailing zero bits): exact product
  constexpr double kLo = 1074.0 * 0x1.a39ef35793c76p-33;  // 1074 * ln2_lo
  const double y = __dadd_rn(__dadd_rn(x, kHi), kLo);
  const double q = fmax(rint(exp(y)), 1.0);  // quanta of 2^-1074; >= 1 on the support
  return __longlong_as_double((long long)q);
}

// K = isinf(C) ? 0 : exp(-C/eps) with C = cost(d2)/scale (geometry.cpp:83-102)
__device__ __forceinline__ double kernel_from_d2(int kind, double d2, double eta, double scale, double eps) {
  const double c = cost_from_d2_rt(kind, d2, eta) / scale;
  return isinf(c) ? 0.0 : exp_ref(-c / eps);
}

template <int KIND>
__device__ __forceinline__ double cost_entry(const double* __restrict__ p, const double* __restrict__ q,
                                             int dim, double eta) {
  double d2 = 0.0;
  for (int k = 0; k < dim; ++k) {
    const double diff = dsub(p[k], q[k]);
    d2 = dadd(d2, dmul(diff, diff));
  }
  if (KIND == 0) return d2;
  if (KIND == 1) return sqrt(d2);
  const double d = sqrt(d2);
  if (d >= dmul(3.14159265358979323846, eta)) return CUDART_INF;
  const double cz = cos(d / dmul(2.0, eta));
  double v = -log(dmul(cz, cz));
  if (!(v >= 0.0)) v = 0.0;
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// std::min(1.0, x) semantics: returns 1.0 when x is NaN (sparsify.cpp:191).
__device__ __forceinline__ double min1(double x) { return (x < 1.0) ? x : 1.0; }

}  // namespace spk
