// shard_core.cuh -- the per-half state machine of the sharded loop, shared by
// the CSR half kernel (shard.cu) and the slab x block one (blocked.cu).
#pragma once

#include "common.cuh"
#include "internal.h"
#include "loop_core.cuh"

#include <memory>

namespace spk {
namespace shard {

constexpr int kT = SPK_SHARD_TAIL;
constexpr int kThreads = 512;
constexpr unsigned long long kNone = ~0ull;

struct State {
  long long t;           // accepted iterations
  long long iterations;  // reported count (includes a failing iteration)
  int stopped, converged, diverged, error_kind, error_half, final_par;
  long long error_index;
  long long masked_rows, masked_cols;
  long long masks_u_pending;
  double err_u_pending;
};

struct HalfArgs {
  int half;       // 0: rows (u from v), 1: columns (v from u)
  int compute;    // 0 = decision only (finish)
  long long t;    // iteration of this half
  int64_t m_own;  // atoms in this rank's slab
  int64_t base;   // global index of slab atom 0
  int64_t m, stride;
  int world;
  long long n, max_iter;
  double delta, exponent;
  int policy;
  const long long* ptr;
  const uint32_t* idx;
  const void* val;
  const double* x;    // gathered input vector (previous half's output, tails inside)
  const double* old;  // own block of the previous iterate of this side
  double* out;        // own block of the new iterate (tail at out + m)
  const double* w;    // own weights (a or b; log weights in the log domain)
  unsigned char* ne;
  int* dyn;
  const State* st_in;
  State* st_out;
  loopcore::Part* part;
  unsigned int* ticket;
  unsigned long long* flag;
};

// The previous half's outcome, from the W tails of the gathered vector x
// (scaling_loop's divergence / ZeroDenominator / mask / stop rules).
template <bool LOG>
__device__ void decide(const HalfArgs& A, State& S) {
  if (S.stopped) return;
  if (A.half == 0 && A.t == 1) return;  // nothing ran before iteration 1
  int rstar = -1;
  double err = 0.0, masks = 0.0, before = 0.0, fidx = 0.0;
  for (int r = 0; r < A.world; ++r) {
    const double* tail = A.x + (int64_t)r * A.stride + A.m;
    if (rstar < 0 && tail[2] > 0.0) {
      rstar = r;
      fidx = tail[2] - 1.0;
      before += tail[3];  // this rank's masks below its first failing atom
    } else if (rstar < 0) {
      before += tail[1];
    }
    err += tail[0];
    masks += tail[1];
  }
  const long long tprev = A.half == 0 ? A.t - 1 : A.t;  // iteration of the half being judged
  const int judged = A.half == 0 ? 1 : 0;               // which half produced x
  if (rstar >= 0) {
    S.stopped = 1;
    S.iterations = tprev;
    if (A.policy == SPK_POLICY_MASK && !LOG) {  // restore the previous iterate (:321-325, :352-356)
      S.diverged = 1;
      S.final_par = (int)((tprev - 1) & 1);
      if (judged == 0) {
        S.masked_rows += (long long)before;
      } else {
        S.masked_rows += S.masks_u_pending;
        S.masked_cols += (long long)before;
      }
    } else {
      S.error_kind = SPK_E_ZERO_DENOMINATOR;
      S.error_half = judged;
      S.error_index = (long long)fidx;
    }
    return;
  }
  if (judged == 0) {  // u-half of iteration t accepted; v-half runs next
    S.masks_u_pending = (long long)masks;
    S.err_u_pending = err;
    return;
  }
  // both halves of iteration tprev accepted
  S.masked_rows += S.masks_u_pending;
  S.masked_cols += (long long)masks;
  S.masks_u_pending = 0;
  S.t = tprev;
  S.iterations = tprev;
  S.final_par = (int)(tprev & 1);
  if (S.masked_rows == A.n || S.masked_cols == A.n) {  // solvers.hpp:357-358 / :465-466
    S.stopped = 1;
    S.error_kind = SPK_E_DEGENERATE_SKETCH_ERROR;
    return;
  }
  if (tprev >= 2 && S.err_u_pending + err <= A.delta) {  // :360-364
    S.stopped = 1;
    S.converged = 1;
    return;
  }
  if (tprev >= A.max_iter) S.stopped = 1;
}

// Reduce this half's (err, masks) over the CTAs: the last CTA to finish
// sums the partials in a fixed order and writes the slab's tail (residual
// partial, dynamic masks, first failing atom + 1, masks before it).
__device__ inline void finish_half(const HalfArgs& A, double err, long long masks) {
  const int lane = threadIdx.x & 31;
  loopcore::block_partial(err, masks, A.part);

  // last CTA to finish reduces the partials in a fixed order and writes the tail
  __shared__ bool last;
  __threadfence();
  if (threadIdx.x == 0) last = atomicAdd(A.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  double e_tot;
  long long m_tot;
  loopcore::reduce_parts(A.part, gridDim.x, e_tot, m_tot);
  const unsigned long long f = __ldcg(A.flag);
  long long before = m_tot;
  if (f != kNone) {  // only masks met before the first failing atom count (:306-307)
    __shared__ long long cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    long long c = 0;
    for (int64_t i = threadIdx.x; i < (int64_t)f; i += blockDim.x) c += (__ldcg(A.dyn + i) == (int)A.t) ? 1 : 0;
    c = warp_sum_ll(c);
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt), (unsigned long long)c);
    __syncthreads();
    before = cnt;
  }
  if (threadIdx.x == 0) {
    double* tail = A.out + A.m;
    tail[0] = e_tot;
    tail[1] = (double)m_tot;
    tail[2] = f == kNone ? 0.0 : (double)(A.base + (int64_t)f) + 1.0;
    tail[3] = (double)before;
    for (int k = 4; k < kT; ++k) tail[k] = 0.0;
    *A.ticket = 0u;
    *A.flag = kNone;
  }
}

// Slab x block half-steps for a shard (blocked.cu): layouts of the shard's
// CSR (rows, columns remapped into the gathered layout) and CSC, and one
// half launched over them. build returns false when the shape does not fit.
struct BlockedShard {
  std::unique_ptr<BlockedHost> R, C;
  DBuf fault;  // [0] first barrier timeout code, [1] its CTA
  int vbytes = 8;
};
bool blocked_shard_build(spk_ctx* ctx, int64_t m_own, int64_t n_in, int64_t nnz_r, const DBuf& row_ptr,
                         const DBuf& col_idx, const DBuf& vals, int64_t nnz_c, const DBuf& col_ptr,
                         const DBuf& row_idx, const DBuf& vals_t, int vbytes, BlockedShard& out);
void blocked_shard_half(spk_ctx* ctx, const HalfArgs& A, BlockedShard& B);

}  // namespace shard
}  // namespace spk
