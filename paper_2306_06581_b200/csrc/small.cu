// small.cu -- the Sinkhorn loop for sketches small enough for shared memory
// (configs 1 and 2: n = 1e3, 1e4): ONE cluster of CS CTAs (up to 16 SMs)
// runs every iteration with no grid barrier.
//
// Reference semantics: detail::scaling_loop (include/sparsink/solvers.hpp:256-395)
// and detail::log_scaling_loop (:397-513), per atom exactly as loop_core.cuh
// (finalize_atom), fast-mode summation (warp per row, FMA / two-pass LSE).
//
// Why: at these sizes the persistent grid loop is bound by its two grid-wide
// barriers per iteration (~10 us per iteration at C1), not by bytes. Here
// every CTA of the cluster keeps BOTH scaling vectors (fp64, full length) in
// its own shared memory, so the gathered x of a half is a shared-memory read.
// A half is split over the CTAs by entry count; each CTA writes the new
// values of its atoms into its own copy and, through DSMEM, into every
// peer's copy; one cluster barrier (hardware, ~1 us less than a grid
// barrier) publishes them with the CTA partials (residual, new masks, first
// failing atom), which every CTA then combines in rank order -- the same
// stop / failure decision everywhere. When the CTA's share of the sketch
// (both halves) also fits, it is staged into shared memory once, and an
// iteration touches no global memory except the per-atom mask state.
// Divergence restore (:321-325, :352-356): each CTA keeps the previous
// iterate of its own atoms and puts it back.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "loop_core.cuh"
#include "rowdot.cuh"

#ifndef SPK_SMALL_WAIT
#define SPK_SMALL_WAIT 0  // 1: test_wait polling, 2: try_wait with a 20 ns suspend hint
#endif

namespace spk {

namespace {

using loopcore::finalize_atom;
using loopcore::kNone;

constexpr int kThreads = 512;  // 16 warps x 4 row groups = 64 rows in flight; 128 registers
constexpr int kMaxCS = 16;

template <class VT>
struct ClusterArgs {
  int64_t n;
  // sketch halves (global); the CTA's share may be staged into shared memory
  const long long* ptr[2];
  const uint32_t* idx[2];
  const VT* val[2];
  int64_t lo[2][kMaxCS + 1];  // atom split of each half by entry count
  const double* w[2];         // a, b (log domain: log a, log b)
  unsigned char* ne[2];       // row / column non-empty flags (dynamic masks)
  int* dyn[2];
  double* out[2];  // final u, v (or log u, log v)
  loopcore::Status* status;
  long long max_iter;
  double delta, exponent;
  int policy;
  long long masked0[2];
  int npad;   // doubles per shared vector
  int stage;  // 1: the CTA's sketch share lives in shared memory
  unsigned long long* trace;  // SPK_TRACE_SMALL=t0: SM clock stamps of iterations t0+1..t0+8 [8][half][rank][kTraceSlots]
  long long trace_t0;
  int64_t stage_ent[2];  // max entries of one CTA's share per half (sliced layout, with padding)
  int64_t stage_rows[2];
  int64_t stage_slices[2];
  // sliced layout of each CTA's share (see group_dot): entry offset of every
  // kSR-row slice, per half, CTAs back to back (CTA r's first slice: soff[h][r])
  const int* sbase[2];
  int64_t soff[2][kMaxCS + 1];
};

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// shared::cluster address of the same shared location in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_cluster(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// bytes of the slab [lo, hi) a CTA sends: lo is even (split_by_entries), the
// end rounded up to even (16-byte bulk copies; the round-up only reaches the
// vector's padding, never another CTA's atoms)
__host__ __device__ __forceinline__ int64_t slab_bytes(int64_t lo, int64_t hi) {
  return hi > lo ? 8 * (((hi + 1) & ~int64_t(1)) - lo) : 0;
}
__device__ __forceinline__ void mbar_init_s(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// bounded wait (a lost transaction must not hang the GPU: the host raises a device error)
__device__ __forceinline__ bool mbar_wait_s(uint64_t* b, uint32_t parity) {
  for (long long spin = 0; spin < (1ll << 26); ++spin) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
#if SPK_SMALL_WAIT == 1
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
#elif SPK_SMALL_WAIT == 2
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 20;\n\t"
#else
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
#endif
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (done) return true;
  }
  return false;
}

template <class T>
__device__ __forceinline__ T* peer(T* p, unsigned rank) {
  T* q;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(q) : "l"(p), "r"(rank));
  return q;
}

#ifndef SPK_SMALL_BULK
#define SPK_SMALL_BULK 1  // 0: slabs as 16-byte st.async per lane (measured slower)
#endif
#ifndef SPK_SMALL_SG
#define SPK_SMALL_SG 4
#endif
constexpr int kSG = SPK_SMALL_SG;  // lanes per row (config-1 rows: ~55 entries)
constexpr int kSR = 32 / kSG;   // rows per warp at once

template <class T>
__device__ __forceinline__ T group_sum(T v) {
#pragma unroll
  for (int o = kSG / 2; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double group_max(double v) {
#pragma unroll
  for (int o = kSG / 2; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One row's dot by the kSG lanes of a group over the sliced share: the
// kSR rows a warp handles at once are stored step-major -- step k of lane l
// at b + 32 k with b = slice base + l -- so every step reads 32 consecutive
// values and indices (no bank conflicts; only the x gather is random).
// `cnt` = this lane's entries of its row. x shared: linear sum of v * x (FMA),
// or the two-pass log-sum-exp (solvers.cpp:99-111; fp32 sketches take the
// fp32-accurate exp). Every lane of the warp must call it.
template <bool LOG, class VT>
__device__ __forceinline__ double group_dot(const VT* val, const uint32_t* idx, int b, int cnt, const double* x) {
  if constexpr (!LOG) {
    double a0 = 0.0, a1 = 0.0;
    int k = 0;
    for (; k + 1 < cnt; k += 2) {
      const int p = b + 32 * k;
      a0 = fma((double)val[p], x[idx[p]], a0);
      a1 = fma((double)val[p + 32], x[idx[p + 32]], a1);
    }
    if (k < cnt) a0 = fma((double)val[b + 32 * k], x[idx[b + 32 * k]], a0);
    return group_sum(a0 + a1);
  } else {
    double m = -CUDART_INF;
    for (int k = 0; k < cnt; ++k) {
      const int p = b + 32 * k;
      const double xv = x[idx[p]];
      if (xv == -CUDART_INF) continue;
      m = fmax(m, log_of(val[p]) + xv);
    }
    m = group_max(m);
    double s = 0.0;
    if (m != -CUDART_INF)
      for (int k = 0; k < cnt; ++k) {
        const int p = b + 32 * k;
        const double xv = x[idx[p]];
        if (xv == -CUDART_INF) continue;
        s += exp_term<VT>(log_of(val[p]) + xv - m);
      }
    s = group_sum(s);
    return m == -CUDART_INF ? -CUDART_INF : m + log(s);
  }
}

constexpr int kTraceSlots = 10;

template <bool LOG, class VT, int CS>
__global__ void __launch_bounds__(kThreads, 1) cluster_loop_kernel(ClusterArgs<VT> A) {
  extern __shared__ __align__(16) double smem[];
  const unsigned rank = CS > 1 ? cluster_rank() : 0u;
  const int64_t n = A.n;
  double* X[2] = {smem, smem + A.npad};  // X[0] = u (rows), X[1] = v (columns)
  // previous iterate of this CTA's own atoms (divergence restore)
  const int64_t own0 = A.lo[0][rank + 1] - A.lo[0][rank], own1 = A.lo[1][rank + 1] - A.lo[1][rank];
  double* prev[2] = {smem + 2 * (int64_t)A.npad, smem + 2 * (int64_t)A.npad + ((own0 + 1) & ~int64_t(1))};
  char* tail = reinterpret_cast<char*>(prev[1] + ((own1 + 1) & ~int64_t(1)));
  // this CTA's atoms' mask state (non-empty flag, dynamic-mask iteration) in
  // shared memory, addressed by the global atom index
  int* dyn_own[2];
  unsigned char* ne_own[2];
  for (int h = 0; h < 2; ++h) {
    const int64_t own = h ? own1 : own0;
    dyn_own[h] = reinterpret_cast<int*>(tail);
    tail += sizeof(int) * ((own + 3) & ~int64_t(3));
  }
  for (int h = 0; h < 2; ++h) {
    const int64_t own = h ? own1 : own0;
    ne_own[h] = reinterpret_cast<unsigned char*>(tail);
    tail += (own + 15) & ~int64_t(15);
  }
  double* w_own[2];
  for (int h = 0; h < 2; ++h) {
    const int64_t own = h ? own1 : own0;
    w_own[h] = reinterpret_cast<double*>(tail);
    tail += sizeof(double) * ((own + 1) & ~int64_t(1));
  }
  const double* w_s[2] = {w_own[0] - A.lo[0][rank], w_own[1] - A.lo[1][rank]};
  unsigned char* ne_s[2] = {ne_own[0] - A.lo[0][rank], ne_own[1] - A.lo[1][rank]};
  int* dyn_s[2] = {dyn_own[0] - A.lo[0][rank], dyn_own[1] - A.lo[1][rank]};
  for (int h = 0; h < 2; ++h)
    for (int64_t i = A.lo[h][rank] + threadIdx.x; i < A.lo[h][rank + 1]; i += blockDim.x) {
      ne_s[h][i] = A.ne[h][i];
      dyn_s[h][i] = 0;
      w_own[h][i - A.lo[h][rank]] = A.w[h][i];
    }
  // the CTA's share of the sketch, staged in shared memory once in the
  // sliced layout (per half: slice bases, row lengths, values, indices);
  // pointers derived from the shared array, so every access is an LDS
  const int* sl[2];
  const int* ln[2];
  const uint32_t* idx[2];
  const VT* val[2];
  for (int h = 0; h < 2; ++h) {
    const int64_t r0 = A.lo[h][rank], r1 = A.lo[h][rank + 1], rows = r1 - r0;
    const int64_t ns = (rows + kSR - 1) / kSR;
    int* ssl = reinterpret_cast<int*>(tail);
    tail += sizeof(int) * ((A.stage_slices[h] + 3) & ~int64_t(3));
    int* sln = reinterpret_cast<int*>(tail);
    tail += sizeof(int) * ((A.stage_rows[h] + 3) & ~int64_t(3));
    VT* sv = reinterpret_cast<VT*>(tail);
    tail += sizeof(VT) * ((A.stage_ent[h] + 3) & ~int64_t(3));
    uint32_t* si = reinterpret_cast<uint32_t*>(tail);
    tail += sizeof(uint32_t) * ((A.stage_ent[h] + 3) & ~int64_t(3));
    const long long* gp = A.ptr[h];
    for (int64_t k = threadIdx.x; k < ns; k += blockDim.x) ssl[k] = A.sbase[h][A.soff[h][rank] + k];
    for (int64_t k = threadIdx.x; k < rows; k += blockDim.x) sln[k] = (int)(gp[r0 + k + 1] - gp[r0 + k]);
    __syncthreads();
    // scatter: row li's entry e goes to step e / kSG of lane (li % kSR) kSG + e % kSG
    for (int64_t li = threadIdx.x >> 5; li < rows; li += blockDim.x >> 5) {
      const int bse = ssl[li / kSR] + (int)(li % kSR) * kSG;
      const long long e0 = gp[r0 + li];
      for (int e = (int)(threadIdx.x & 31); e < sln[li]; e += 32) {
        const int dst = bse + (e / kSG) * 32 + (e % kSG);
        sv[dst] = A.val[h][e0 + e];
        si[dst] = A.idx[h][e0 + e];
      }
    }
    sl[h] = ssl;
    ln[h] = sln;
    idx[h] = si;
    val[h] = sv;
  }
  __shared__ double scratch[32];
  __shared__ int mscratch[32];
  __shared__ double comb_e[2];  // per half: the cluster's combined partials
  __shared__ long long comb_m[2];
  __shared__ unsigned long long comb_f[2];
  __shared__ unsigned long long flag_sh[2];
  // per half: every peer's partials {residual (lo, hi), masks, first failing
  // atom or ~0}, slot = its rank (the own slot stays in registers)
  static_assert(CS <= kThreads / 32, "one sending warp per peer");
  __shared__ uint4 xs[2][CS];
  __shared__ __align__(8) uint64_t mbar[2];  // per half: the peers' st.async bytes
  __shared__ unsigned long long trace_sh[8 * 2 * kTraceSlots];  // SPK_TRACE_SMALL stamps, copied out at the end
  if (A.trace)
    for (int k = threadIdx.x; k < 8 * 2 * kTraceSlots; k += blockDim.x) trace_sh[k] = 0ull;
  const double on = LOG ? 0.0 : 1.0, off = LOG ? -CUDART_INF : 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {  // u = v = 1 on covered atoms (:277-281, :424-428)
    X[0][i] = A.ne[0][i] ? on : off;
    X[1][i] = A.ne[1][i] ? on : off;
  }
  if (threadIdx.x == 0) {
    flag_sh[0] = flag_sh[1] = kNone;
    mbar_init_s(&mbar[0]);
    mbar_init_s(&mbar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // bytes each half receives from the peers: their atoms' new values + their
  // partials (residual, masks, first failing atom)
  uint32_t rx_bytes[2] = {0u, 0u};
  for (int h = 0; h < 2; ++h)
    for (int r = 0; r < CS; ++r)
      if (r != (int)rank) rx_bytes[h] += (uint32_t)(slab_bytes(A.lo[h][r], A.lo[h][r + 1]) + 16);
  if (CS > 1) cluster_barrier();  // peers' vectors and barriers initialised before any remote store
  else __syncthreads();
  unsigned long long clock0 = 0;  // SPK_TRACE_SMALL: common origin of the CTAs' clocks
  if (A.trace) asm volatile("mov.u64 %0, %%clock64;" : "=l"(clock0));

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5, gl = lane & (kSG - 1);
  const bool need_err = A.delta >= 0.0;  // eu + ev <= delta can only hold for delta >= 0
  long long mr = A.masked0[0], mc = A.masked0[1];
  long long t = 0;
  int converged = 0, diverged = 0, ekind = 0, ehalf = 0, dhalf = 0;
  long long eidx = 0, didx = 0, mr_before = mr, mc_before = mc, mu_last = 0;
  uint32_t parity = 0u;  // bit h: phase parity of mbar[h] to wait for next
  bool faulted = false;  // a peer transfer never completed (reported, never hangs)

  // one half: h = 0 rows against v (u-half), h = 1 columns against the new u.
  // Every new value goes to the peers as st.async (remote shared store that
  // completes a transaction count on the RECEIVER's mbarrier), and so do the
  // CTA's partials: a CTA proceeds once its mbarrier has seen every byte of
  // the half from every peer -- no cluster barrier, no release fence. Reuse is
  // safe: a peer can only start writing this half's vector again after it has
  // received all of this CTA's values of the following half, i.e. after this
  // CTA stopped reading it.
  auto stamp = [&](int h, int k) {
    if (A.trace && t > A.trace_t0 && t <= A.trace_t0 + 8 && threadIdx.x == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(g));
      trace_sh[((t - 1 - A.trace_t0) * 2 + h) * kTraceSlots + k] = g - clock0;  // shared: no global store in flight
      // (%globaltimer reads cost ~0.5 us each here: SM clocks only, aligned
      // across the cluster by the clock each CTA read leaving the first cluster barrier)
    }
  };
  auto half = [&](int h, double& err_all, long long& masks_all, unsigned long long& flag_all) {
    stamp(h, 0);
    if (CS > 1 && threadIdx.x == 0) mbar_expect_tx(&mbar[h], rx_bytes[h]);
    const int64_t r0 = A.lo[h][rank], r1 = A.lo[h][rank + 1];
    const double* x = X[h ^ 1];
    double* out = X[h];
    const uint32_t bar_h = smem_u32(&mbar[h]);
    double err = 0.0;
    long long masks = 0;
    // kSG lanes per row, kSR rows per warp at once: every row of a config-1
    // slab is in flight in one pass
    for (int64_t i0 = r0 + (int64_t)warp * kSR; i0 < r1; i0 += (int64_t)nw * kSR) {
      const int64_t i = i0 + lane / kSG;
      const bool in = i < r1;
      const double old = in ? out[i] : 0.0;
      if (in && gl == 0) prev[h][i - r0] = old;
      const bool live = in && ne_s[h][i];  // structurally empty / masked: keeps its value
      int b = 0, cnt = 0;  // lane's first staged entry (a share holds < 2^31), its entry count
      if (live) {
        const int li = (int)(i - r0), len = ln[h][li];
        b = sl[h][li / kSR] + lane;
        cnt = len > gl ? (len - gl + kSG - 1) / kSG : 0;
      }
      const double tmp = group_dot<LOG, VT>(val[h], idx[h], b, cnt, x);
      if (live && gl == 0)
        err += finalize_atom<LOG>(i, tmp, old, w_s[h][i], A.exponent, A.policy, (int)t, ne_s[h], dyn_s[h], out,
                                  &flag_sh[h], masks);
    }
    // the residual only feeds the delta stop: no reductions when it is off
    if (need_err) err = warp_sum(err);
    const int wm = (int)__reduce_add_sync(0xffffffffu, (unsigned)masks);
    if (lane == 0) {
      scratch[warp] = err;
      mscratch[warp] = wm;
    }
    __syncthreads();
    stamp(h, 1);
    // CTA partials (fixed shuffle tree: every warp gets the same values) and
    // the transfers: warp w serves peer w -- ONE bulk copy of this CTA's slab
    // of the new vector (shared -> peer shared, completing bytes on the peer's
    // mbarrier; the fence makes the CTA's generic stores visible to the async
    // proxy) and ONE 16-byte st.async of the partials on the same mbarrier.
    double own_e = 0.0;
    int own_m = 0;
    unsigned own_f = 0xffffffffu;
    if (warp < CS) {
      double e = (need_err && lane < nw) ? scratch[lane] : 0.0;
      if (need_err) e = warp_sum(e);
      const int m = (int)__reduce_add_sync(0xffffffffu, lane < nw ? (unsigned)mscratch[lane] : 0u);
      const unsigned long long f64 = flag_sh[h];
      const unsigned f = f64 == kNone ? 0xffffffffu : (unsigned)f64;  // atom index < 2^31
      stamp(h, 8);
      if (warp == 0) {  // the combining warp keeps the CTA's own slot in registers
        own_e = e;
        own_m = m;
        own_f = f;
      }
      if (warp != (int)rank) {
        const uint32_t pr = (uint32_t)warp, rb = map_cluster(bar_h, pr);
        const uint32_t bytes = (uint32_t)slab_bytes(r0, r1);
#if SPK_SMALL_BULK
        if (lane == 0 && bytes) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          stamp(h, 9);
          const uint32_t src = smem_u32(out + r0);
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  map_cluster(src, pr)),
              "r"(src), "r"(bytes), "r"(rb)
              : "memory");
        }
#else
        // the slab as 16-byte remote stores, one per lane and step (the TMA
        // path serialises the CTA's CS - 1 small bulk copies: ~1.7 us a half)
        const uint32_t dst = map_cluster(smem_u32(out + r0), pr);
        const uint4* src = reinterpret_cast<const uint4*>(out + r0);
        for (uint32_t c = (uint32_t)lane; c < bytes / 16u; c += 32u) {
          const uint4 v = src[c];
          asm volatile(
              "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                  dst + 16u * c),
              "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rb)
              : "memory");
        }
#endif
        if (lane == 0)
          asm volatile(
              "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                  map_cluster(smem_u32(&xs[h][rank]), pr)),
              "r"((unsigned)__double2loint(e)), "r"((unsigned)__double2hiint(e)), "r"((unsigned)m), "r"(f), "r"(rb)
              : "memory");
      }
    }
    stamp(h, 2);
    // every peer's values and partials of this half have landed: one warp
    // waits (CTA-scope acquire: the data is in this CTA's shared memory; a
    // cluster-scope acquire would invalidate L1 on every poll), the barrier
    // below publishes the completion -- and this CTA's own stores -- to all
    // The same warp then combines the CS slots (a fixed butterfly over lanes
    // 0..CS-1: identical sums on every CTA) and publishes them with the barrier.
    if (warp == 0) {
      if (CS > 1 && !mbar_wait_s(&mbar[h], (parity >> h) & 1u)) faulted = true;
      const uint4 sl = (lane < CS && lane != (int)rank) ? xs[h][lane] : make_uint4(0u, 0u, 0u, 0xffffffffu);
      double e = lane == (int)rank ? own_e : need_err ? __hiloint2double((int)sl.y, (int)sl.x) : 0.0;
      int m = lane == (int)rank ? own_m : (int)sl.z;
      unsigned f = lane == (int)rank ? own_f : sl.w;
#pragma unroll
      for (int o = 1; o < CS; o <<= 1) {
        if (need_err) e += __shfl_xor_sync(0xffffffffu, e, o);
        m += __shfl_xor_sync(0xffffffffu, m, o);
        f = min(f, __shfl_xor_sync(0xffffffffu, f, o));
      }
      if (lane == 0) {
        comb_e[h] = e;
        comb_m[h] = m;
        comb_f[h] = f == 0xffffffffu ? kNone : (unsigned long long)f;
      }
    }
    parity ^= 1u << h;
    __syncthreads();
    stamp(h, 3);
    if (threadIdx.x == 0) flag_sh[h] = kNone;  // every warp has read it: recycled for the next pass of this half
    err_all = comb_e[h];
    masks_all = comb_m[h];
    flag_all = comb_f[h];
    stamp(h, 4);
  };
  auto restore = [&](int h) {  // previous iterate of this CTA's atoms (every CTA restores its own)
    const int64_t r0 = A.lo[h][rank], r1 = A.lo[h][rank + 1];
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) X[h][i] = prev[h][i - r0];
  };

  while (t < A.max_iter) {
    ++t;
    mr_before = mr;
    mc_before = mc;
    double eu, ev;
    long long mu, mv;
    unsigned long long fu, fv;
    half(0, eu, mu, fu);
    if (__syncthreads_or(faulted)) break;
    if (fu != kNone) {
      if (A.policy == SPK_POLICY_MASK && !LOG) {
        diverged = 1;
        dhalf = 0;
        didx = (long long)fu;
      } else {
        ekind = SPK_E_ZERO_DENOMINATOR;
        ehalf = 0;
        eidx = (long long)fu;
      }
      restore(0);
      mu_last = 0;
      break;
    }
    half(1, ev, mv, fv);
    if (__syncthreads_or(faulted)) break;
    if (fv != kNone) {
      if (A.policy == SPK_POLICY_MASK && !LOG) {
        diverged = 1;
        dhalf = 1;
        didx = (long long)fv;
      } else {
        ekind = SPK_E_ZERO_DENOMINATOR;
        ehalf = 1;
        eidx = (long long)fv;
      }
      restore(0);
      restore(1);
      mu_last = mu;
      break;
    }
    mr += mu;
    mc += mv;
    if (mr == n || mc == n) {  // solvers.hpp:357-358 / :465-466
      ekind = SPK_E_DEGENERATE_SKETCH_ERROR;
      break;
    }
    if (t >= 2 && eu + ev <= A.delta) {
      converged = 1;
      break;
    }
  }
  __syncthreads();
  for (int h = 0; h < 2; ++h)  // each CTA stores its own atoms (and their dynamic-mask stamps)
    for (int64_t i = A.lo[h][rank] + threadIdx.x; i < A.lo[h][rank + 1]; i += blockDim.x) {
      A.out[h][i] = X[h][i];
      A.dyn[h][i] = dyn_s[h][i];
    }
  if (A.trace)
    for (int k = threadIdx.x; k < 8 * 2 * kTraceSlots; k += blockDim.x)
      A.trace[((k / kTraceSlots) * CS + rank) * kTraceSlots + k % kTraceSlots] = trace_sh[k];
  if (CS > 1) cluster_barrier();  // no CTA leaves while a peer may still read its Xch
  if (threadIdx.x == 0 && rank == 0) {
    loopcore::Status* s = A.status;
    s->iterations = t;
    s->converged = converged;
    s->diverged = diverged;
    s->error_kind = faulted ? SPK_E_DEVICE : ekind;
    s->error_half = ehalf;
    s->error_index = eidx;
    s->cur = 0;
    s->div_half = dhalf;
    s->div_index = didx;
    s->masked_rows_before = mr_before;
    s->masked_cols_before = mc_before;
    s->masks_u_last = mu_last;
    s->masked_rows = mr;
    s->masked_cols = mc;
  }
}

// Atom split of a half over CS CTAs by entry count (host copy of ptr).
void split_by_entries(const std::vector<long long>& ptr, int64_t n, int CS, int64_t* lo) {
  const long long total = ptr[n];
  lo[0] = 0;
  for (int r = 1; r < CS; ++r) {
    const long long target = (long long)((double)total * r / CS);
    lo[r] = std::lower_bound(ptr.begin(), ptr.begin() + n + 1, target) - ptr.begin();
    lo[r] = std::min<int64_t>(n, (lo[r] + 1) & ~int64_t(1));  // even: 16-byte aligned slabs (bulk copies)
    lo[r] = std::max(lo[r], lo[r - 1]);
  }
  lo[CS] = n;
}

template <bool LOG, class VT, int CS>
bool launch_cluster(spk_ctx* ctx, ClusterArgs<VT>& A, size_t smem) {
  auto kern = cluster_loop_kernel<LOG, VT, CS>;
  loopcore::allow_max_dyn_smem((const void*)kern);
  if (CS > 8) SPK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(CS);
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)kern, &lc) != cudaSuccess || nclusters < 1) {
    (void)cudaGetLastError();
    return false;
  }
  void* args[] = {&A};
  SPK_CUDA(cudaLaunchKernelExC(&lc, (const void*)kern, args));
  return true;
}

template <bool LOG, class VT>
bool run_cluster_t(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy,
                   LoopState& st, LoopOut& out) {
  const int64_t n = sk->n;
  int optin = 0;
  SPK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const size_t budget = (size_t)optin - 4096;  // static shared use
  const int npad = (int)((n + 31) & ~int64_t(31));
  std::vector<long long> rp(n + 1), cp(n + 1);
  download(ctx, rp.data(), sk->row_ptr, sizeof(long long) * (n + 1));
  download(ctx, cp.data(), sk->col_ptr, sizeof(long long) * (n + 1));
  ClusterArgs<VT> A{};
  int CS = 0;
  size_t smem = 0;
  std::vector<int> sb[2];  // slice bases of the chosen split
  for (int cs : {ctx->small_cluster, 8, 4, 2, 1}) {  // largest cluster first; stage the sketch when it fits
    if (cs < 1 || cs > kMaxCS || (cs & (cs - 1))) continue;
    ClusterArgs<VT> B{};
    split_by_entries(rp, n, cs, B.lo[0]);
    split_by_entries(cp, n, cs, B.lo[1]);
    int64_t own[2] = {0, 0}, ent[2] = {0, 0}, nsl[2] = {0, 0};
    std::vector<int> bases[2];
    for (int h = 0; h < 2; ++h) {
      const std::vector<long long>& p = h ? cp : rp;
      for (int r = 0; r < cs; ++r) {
        const int64_t r0 = B.lo[h][r], r1 = B.lo[h][r + 1];
        own[h] = std::max(own[h], r1 - r0);
        B.soff[h][r] = (int64_t)bases[h].size();
        int64_t acc = 0;  // padded entries of the share: every slice takes its longest row's steps x 32
        for (int64_t s0 = r0; s0 < r1; s0 += kSR) {
          long long steps = 0;
          for (int64_t i = s0; i < std::min(r1, s0 + kSR); ++i) steps = std::max(steps, (p[i + 1] - p[i] + kSG - 1) / kSG);
          bases[h].push_back((int)acc);
          acc += 32 * steps;
        }
        ent[h] = std::max(ent[h], acc);
        nsl[h] = std::max<int64_t>(nsl[h], (int64_t)bases[h].size() - B.soff[h][r]);
      }
      B.soff[h][cs] = (int64_t)bases[h].size();
    }
    size_t base = sizeof(double) * (2 * (size_t)npad + ((own[0] + 1) & ~1) + ((own[1] + 1) & ~1));
    for (int h = 0; h < 2; ++h)
      base += sizeof(int) * ((own[h] + 3) & ~3) + ((own[h] + 15) & ~15) + sizeof(double) * ((own[h] + 1) & ~1);
    size_t staged = 0;
    for (int h = 0; h < 2; ++h)
      staged += sizeof(int) * (((nsl[h] + 3) & ~3) + ((own[h] + 3) & ~3)) + (sizeof(VT) + 4) * ((ent[h] + 3) & ~3);
    // the cluster's SMs win only while the sketch lives in their shared memory:
    // streamed from L2 by <= 16 SMs it loses to the whole-GPU grid loop
    if (ent[0] >= (1ll << 31) || ent[1] >= (1ll << 31) || base + staged > budget) continue;
    B.stage = 1;
    for (int h = 0; h < 2; ++h) {
      B.stage_ent[h] = ent[h];
      B.stage_rows[h] = own[h];
      B.stage_slices[h] = nsl[h];
      sb[h] = std::move(bases[h]);
    }
    smem = base + staged;
    A = B;
    CS = cs;
    break;
  }
  if (!CS) return false;

  LoopWs& W = sk->ws;
  W.row_ne.ensure(n);
  W.col_ne.ensure(n);
  W.dyn_row.ensure(sizeof(int) * n);
  W.dyn_col.ensure(sizeof(int) * n);
  W.u2.ensure(sizeof(double) * (2 * (size_t)npad + 16));
  W.status.ensure(sizeof(loopcore::Status));
  cudaStream_t s = ctx->stream;
  SPK_CUDA(cudaMemcpyAsync(W.row_ne.p, sk->cov_row.p, n, cudaMemcpyDeviceToDevice, s));
  SPK_CUDA(cudaMemcpyAsync(W.col_ne.p, sk->cov_col.p, n, cudaMemcpyDeviceToDevice, s));
  SPK_CUDA(cudaMemsetAsync(W.dyn_row.p, 0, sizeof(int) * n, s));
  SPK_CUDA(cudaMemsetAsync(W.dyn_col.p, 0, sizeof(int) * n, s));
  SPK_CUDA(cudaMemsetAsync(W.status.p, 0, sizeof(loopcore::Status), s));
  const double* wa = st.a;
  const double* wb = st.b;
  if (LOG) {
    W.la.ensure(sizeof(double) * n);
    W.lb.ensure(sizeof(double) * n);
    loopcore::log_weights_kernel<<<loopcore::simple_grid(ctx, n), 256, 0, s>>>(n, st.a, W.la.as<double>());
    loopcore::log_weights_kernel<<<loopcore::simple_grid(ctx, n), 256, 0, s>>>(n, st.b, W.lb.as<double>());
    ctx->launches += 2;
    wa = W.la.as<double>();
    wb = W.lb.as<double>();
  }
  A.n = n;
  A.ptr[0] = sk->row_ptr.as<long long>();
  A.ptr[1] = sk->col_ptr.as<long long>();
  A.idx[0] = sk->col_idx.as<uint32_t>();
  A.idx[1] = sk->row_idx.as<uint32_t>();
  if constexpr (std::is_same<VT, LogK>::value || std::is_same<VT, LogKf>::value) {
    A.val[0] = reinterpret_cast<const VT*>(sk->log_values.p);
    A.val[1] = reinterpret_cast<const VT*>(sk->log_values_t.p);
  } else {
    A.val[0] = sk->values.as<VT>();
    A.val[1] = sk->values_t.as<VT>();
  }
  A.w[0] = wa;
  A.w[1] = wb;
  A.ne[0] = W.row_ne.as<unsigned char>();
  A.ne[1] = W.col_ne.as<unsigned char>();
  A.dyn[0] = W.dyn_row.as<int>();
  A.dyn[1] = W.dyn_col.as<int>();
  A.out[0] = W.u2.as<double>();
  A.out[1] = W.u2.as<double>() + npad;
  A.status = W.status.as<loopcore::Status>();
  A.max_iter = cfg.max_iter;
  A.delta = cfg.delta;
  A.exponent = exponent;
  A.policy = policy;
  A.masked0[0] = sk->cov_empty_rows;
  A.masked0[1] = sk->cov_empty_cols;
  A.npad = npad;
  {  // slice bases of both halves in one buffer
    std::vector<int> all(sb[0]);
    all.insert(all.end(), sb[1].begin(), sb[1].end());
    upload(ctx, W.slices, all.data(), sizeof(int) * all.size());
    A.sbase[0] = W.slices.as<int>();
    A.sbase[1] = W.slices.as<int>() + sb[0].size();
  }
  DBuf trace;
  const bool tracing = std::getenv("SPK_TRACE_SMALL") != nullptr;
  if (tracing) A.trace_t0 = std::max(0ll, std::atoll(std::getenv("SPK_TRACE_SMALL")));
  if (tracing) {
    trace.alloc(sizeof(unsigned long long) * 8 * 2 * kMaxCS * kTraceSlots);
    SPK_CUDA(cudaMemsetAsync(trace.p, 0, trace.bytes, s));
    A.trace = trace.as<unsigned long long>();
  }
  Timer tm(s);
  bool ok = false;
  switch (CS) {
    case 16: ok = launch_cluster<LOG, VT, 16>(ctx, A, smem); break;
    case 8: ok = launch_cluster<LOG, VT, 8>(ctx, A, smem); break;
    case 4: ok = launch_cluster<LOG, VT, 4>(ctx, A, smem); break;
    case 2: ok = launch_cluster<LOG, VT, 2>(ctx, A, smem); break;
    default: ok = launch_cluster<LOG, VT, 1>(ctx, A, smem); break;
  }
  if (!ok) return false;
  ++ctx->launches;
  out.loop_s = tm.stop();
  SPK_CUDA(cudaGetLastError());
  loopcore::Status S;
  download(ctx, &S, W.status, sizeof S);
  if (S.error_kind == SPK_E_DEVICE) fail_device("small loop: a peer's st.async transfer timed out", cudaErrorLaunchTimeout);
  if (tracing) {  // per-phase mean SM cycles over iterations 2..8 (thread 0 of every CTA)
    std::vector<unsigned long long> tr(8 * 2 * kMaxCS * kTraceSlots);
    download(ctx, tr.data(), trace, sizeof(unsigned long long) * tr.size());
    double ph[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    int cnt9 = 0;
    int cnt = 0;
    for (int it = 1; it < 8 && it + A.trace_t0 < S.iterations; ++it)
      for (int h = 0; h < 2; ++h)
        for (int r = 0; r < CS; ++r) {
          const unsigned long long* q = &tr[(((size_t)it * 2 + h) * CS + r) * kTraceSlots];
          for (int k = 0; k < 4; ++k) ph[k] += (double)(q[k + 1] - q[k]);
          ph[8] += (double)(q[8] - q[1]);  // CTA partial reductions
          if (q[9]) {
            ph[9] += (double)(q[9] - q[8]);  // proxy fence
            ++cnt9;
          }
          ++cnt;
        }
    for (int h = 0; h < 2; ++h) {  // per-rank row pass and stamp-0 skew (iterations 2..8)
      std::fprintf(stderr, "SPK_TRACE_SMALL half %d rows/start-skew per rank:", h);
      for (int r = 0; r < CS; ++r) {
        double rows = 0, skew = 0;
        int c = 0;
        for (int it = 1; it < 8 && it + A.trace_t0 < S.iterations; ++it, ++c) {
          const unsigned long long* q = &tr[(((size_t)it * 2 + h) * CS + r) * kTraceSlots];
          rows += (double)(q[1] - q[0]);
          skew += (double)(q[3] - q[2]);
        }
        if (c) std::fprintf(stderr, " %.0f/%.0f", rows / c, skew / c);
      }
      std::fprintf(stderr, "\n");
    }
    for (int h = 0; h < 2; ++h) {  // cluster timeline of one half (cycles after the earliest start), iterations 2..8
      std::fprintf(stderr, "SPK_TRACE_SMALL half %d timeline per rank [start rows-done sent peers-in combined]:", h);
      for (int r = 0; r < CS; ++r) {
        double ph2[5] = {0, 0, 0, 0, 0};
        int c = 0;
        for (int it = 1; it < 8 && it + A.trace_t0 < S.iterations; ++it, ++c) {
          unsigned long long t0 = ~0ull;
          for (int r2 = 0; r2 < CS; ++r2) t0 = std::min(t0, tr[(((size_t)it * 2 + h) * CS + r2) * kTraceSlots]);
          const unsigned long long* q = &tr[(((size_t)it * 2 + h) * CS + r) * kTraceSlots];
          for (int k = 0; k < 5; ++k) ph2[k] += (double)(q[k] - t0);
        }
        if (c) std::fprintf(stderr, " r%d[%.0f %.0f %.0f %.0f %.0f]", r, ph2[0] / c, ph2[1] / c, ph2[2] / c, ph2[3] / c, ph2[4] / c);
      }
      std::fprintf(stderr, "\n");
    }
    if (cnt)
      std::fprintf(stderr,
                   "SPK_TRACE_SMALL CS=%d (cycles): rows %.0f, partials %.0f [reduce %.0f fence %.0f], peer wait %.0f, "
                   "combine %.0f\n",
                   CS, ph[0] / cnt, ph[1] / cnt, ph[8] / cnt, cnt9 ? ph[9] / cnt9 : 0.0, ph[2] / cnt, ph[3] / cnt);
  }
  loopcore::loop_epilogue<LOG>(ctx, S, n, W, A.out[0], A.out[1], st, out);
  return true;
}

}  // namespace

// Fast-mode loop on one cluster when the sketch is small enough (both
// scaling vectors in every CTA's shared memory). Returns false when it does
// not apply (the caller then runs the grid loop).
bool run_cluster_loop(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy,
                      LoopState& st, LoopOut& out) {
  if (ctx->deterministic || !ctx->small_loop || sk->n_cols) return false;
  if (sk->n > ctx->small_max_n || sk->nnz > ctx->small_max_nnz) return false;
  // the loop's entry checks (solvers.hpp:269-274 / :411-414) are the grid loop's: let it raise them
  if ((sk->cov_empty_rows || sk->cov_empty_cols) && policy == SPK_POLICY_ERROR) return false;
  if (sk->cov_empty_rows == sk->n || sk->cov_empty_cols == sk->n) return false;
  const bool log_domain = cfg.stabilize != 0;
  if (log_domain) {
    ensure_log_values(ctx, sk);
    if (sk->value_type == SPK_VALUES_F32) return run_cluster_t<true, LogKf>(ctx, sk, cfg, exponent, policy, st, out);
    return run_cluster_t<true, LogK>(ctx, sk, cfg, exponent, policy, st, out);
  }
  if (sk->value_type == SPK_VALUES_F32) return run_cluster_t<false, float>(ctx, sk, cfg, exponent, policy, st, out);
  return run_cluster_t<false, double>(ctx, sk, cfg, exponent, policy, st, out);
}

}  // namespace spk
