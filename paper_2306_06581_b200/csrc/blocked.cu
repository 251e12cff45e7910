// blocked.cu -- the fast sparse half-step: slab x block sketch layout with the
// scaling vector staged in shared memory by TMA (north-star item 3:
// "shared-memory/TMA staging of the gathered scaling vector").
//
// Why: at config 4 (n = 1e6, 1.1e8 entries, columns uniformly random) every
// gathered x[j] of the CSR kernel is a random 8-byte read, i.e. one 32-byte L2
// sector per entry: 3.5 GB of L2->SM sectors per half on top of the 0.9 GB
// entry stream (profiles/r1_c4_csr_loop_ncu.json: 9.5 GB L2 reads/iteration).
//
// Layout (built once per sketch, for the CSR and for the CSC mirror):
//   output atoms (this half's rows) are cut into Q row slabs of ~equal entry
//   count; each slab is served by S CTAs (S = 2: a CTA pair, each reading
//   one half of x -- equal halves -- so every SM stages n/2 instead of n
//   scalings per half); a CTA's columns are cut into blocks of W <= 4096
//   atoms (one 32 KB x tile). Inside a CTA the slab's rows are cut into 15
//   warp ranges of ~equal entry count. Entries are ordered (CTA, warp, block,
//   chunk): each warp's half is ONE contiguous stream of 32-entry chunks,
//   every chunk holding 32 DISTINCT rows (so lanes add into shared
//   accumulators without atomics). Which entries of a (warp, block) segment
//   share a chunk is chosen by color_warp_kernel so that a half-warp's 16
//   accumulators and its 16 gathered x lie in 16 different bank pairs wherever
//   the segment allows. A row's entries are therefore summed chunk by chunk,
//   not in column order (sparsify.cpp:203-226 order is the CSR loop's and the
//   deterministic mode's; this fast mode agrees with it to ~5e-15).
//   Entries are packed (row_local << 16 | new-block flag << 12 | col_local)
//   + value; the first chunk of every block carries the flag, so the loop
//   reads no per-block offsets; four consecutive chunks are interleaved per
//   lane, so one 16-byte load gives a lane its entries of 4 chunks: the
//   stream goes HBM -> registers directly. Padding (value 0) adds into 16
//   sink rows behind the slab's accumulators.
// Half-step (inside the persistent loop, loop_core.cuh), 16 warps per CTA:
//   * producer warp: cp.async.bulk (TMA) of the CTA's x tiles through a
//     STG-deep ring (full/empty mbarriers);
//   * 15 consumer warps stream their entries with coalesced 16-byte loads in
//     two register sets of kDepth groups (one is folded while the other is in
//     flight), evict-first in L2 (the stream never fits; x must stay), gather
//     x from the shared tile and add v * x into their rows' fp64 shared
//     accumulators;
//   * S = 2: the pair is a 2-CTA cluster and each CTA finalizes half of the
//     slab as p0 + p1, reading the partner's sums over DSMEM (or swapping them
//     through L2 when the pairs cannot be co-scheduled as clusters).
// L2->SM traffic per half: the entry stream + Q * n * 8 bytes of x tiles.
// DESIGN.md section 4.1 has the measurements behind each of these choices.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "internal.h"
#include "loop_core.cuh"
#include "shard_core.cuh"

namespace spk {

namespace {

#ifndef SPK_NW
#define SPK_NW 15  // variant builds (profiling): 7 and 11 consumer warps measured slower, DESIGN.md section 4.1
#endif
constexpr int kNW = SPK_NW;             // consumer warps per CTA (+1 producer = 16 warps: 4 per SMSP, 128 registers)
constexpr int kThreadsBlocked = 32 * (kNW + 1);
constexpr int kTileW = 4096;            // x tile: 32 KB of fp64
constexpr int kGE = 128;                // entries per group (4 chunks; one 16-byte load per lane)
// Packed key of an entry: row_local << 16 | kNewBlock? | col_local, bits 13-15
// zero (so key >> 13 is the byte offset of the row's fp64 accumulator).
constexpr uint32_t kNewBlock = 0x1000u;  // this chunk is the first of the next column block
constexpr uint32_t kColMask = 0x0fffu;
// Padding entries (value 0) add into sink rows max_rows .. max_rows + 15 of the half: one per bank pair, so a
// pad can take a bank class its half-chunk does not use.
constexpr int kSinkRows = 16;

// ---- PTX helpers: mbarrier + 1-D bulk copy (TMA) ------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Bounded wait: false after ~2^20 polls (a lost transaction must not hang the
// GPU; the caller records a fault and the host raises it). The fault word is
// only read once a poll has failed (every 256th poll), so a wait on an
// already-complete phase costs no global load; after a fault, waits drain fast.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __noinline__ bool mbar_wait_slow(uint64_t* bar, uint32_t parity, const unsigned int* fault) {
  for (int spin = 0; spin < (1 << 20); ++spin) {
    if ((spin & 255) == 0 && __ldcg(fault)) return false;
    if (mbar_try(bar, parity)) return true;
  }
  return false;
}
__device__ __forceinline__ bool mbar_wait(uint64_t* bar, uint32_t parity, const unsigned int* fault) {
  return mbar_try(bar, parity) || mbar_wait_slow(bar, parity, fault);
}
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 16-byte global -> shared copy (Ampere-style cp.async, L2 only), grouped per thread.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// wait until at most N of this thread's groups are pending
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Shared-memory fp64 accesses by 32-bit shared address: the accumulator and
// tile bases stay in registers (the generic-pointer form re-derived the
// shared window base, an S2UR and its wait, for every chunk).
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

__device__ __forceinline__ void record_fault(unsigned int* fault, unsigned int code) {
  if (atomicCAS(fault, 0u, code) == 0u) fault[1] = blockIdx.x;
}

// Streaming 16-byte load of the entry stream: read-only, no L1 allocation,
// evict-first in L2 (the 1.8 GB stream must not push the scalings out).
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ldg_stream(const void* p, uint64_t pol) {
  uint4 r;
#if defined(SPK_LDPOL) && SPK_LDPOL == 1  // variant builds (profiling): no L2 policy
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
#elif defined(SPK_LDPOL) && SPK_LDPOL == 2  // L1 allocating, evict-first
  asm("ld.global.nc.L1::evict_first.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
#else
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
#endif
  return r;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Cluster barrier with release/acquire semantics (shared::cluster writes of
// each CTA visible to the other after it) and the peer's view of a shared address.
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ const double* map_peer(const double* p, unsigned rank) {
  const double* q;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(q) : "l"(p), "r"(rank));
  return q;
}

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Stream position of (global chunk C, lane) -- 4-chunk groups interleaved per lane.
__host__ __device__ __forceinline__ int64_t pos_packed(int64_t C, int lane) {
  return (C >> 2) * kGE + 4 * lane + (C & 3);
}
__host__ __device__ __forceinline__ int64_t pos_f64(int64_t C, int lane) {
  return (C >> 2) * kGE + ((C & 3) >> 1) * 64 + 2 * lane + (C & 1);
}

template <class VT>
struct Group {  // one lane's entries of 4 consecutive chunks
  uint4 k;
  uint4 v0;
  uint4 v1;  // f64 only
};

// CL: the CTA pair is a 2-CTA cluster and reads the partner's partial sums
// from its shared memory (DSMEM) instead of swapping them through L2.
template <class VT, int S, int STG, bool CL = false>
struct BlockedOp {
  static constexpr int kThreads = kThreadsBlocked;
  static constexpr int kCluster = CL ? 2 : 1;
  static constexpr int kMinBlocks = 1;  // one CTA per SM: full register file, up to 227 KB shared
#ifdef SPK_DEPTH
  static constexpr int kDepth = SPK_DEPTH;
#else
  // groups per register set (two sets per consumer warp). Measured at config 4
  // (f32): 1 -> 1960, 2 -> 2579, 3 -> 2368, 4 -> 2210 iterations/s: a deeper
  // set unrolls more copies of the group code (instruction cache) for no gain
  // in bytes in flight that matters.
  static constexpr int kDepth = 2;
#endif
  BlockedHalf L[2];
  int64_t n;
  int acc_rows;         // shared accumulator capacity (max rows of a slab over both halves)
  unsigned int* fault;  // [0] first fault code, [1] its CTA
  double* xchg;         // S = 2: partial sums handed to the partner CTA (n doubles)
  unsigned int* pair;   // S = 2: one arrival counter per row slab
  unsigned long long* trace;  // SPK_TRACE_BLOCKED: globaltimer stamps of the first 4 iterations
  bool fresh;                 // one launch per half (sharded): initialise the barriers on every call

  __host__ __device__ size_t head_bytes() const { return align16((size_t)(acc_rows + kSinkRows) * 8) + 128; }
  size_t smem_bytes() const { return head_bytes() + (size_t)STG * kTileW * 8; }

  __device__ __forceinline__ static double value(const Group<VT>& g, int k) {
    if (sizeof(VT) == 4) {
      const uint32_t b = k == 0 ? g.v0.x : k == 1 ? g.v0.y : k == 2 ? g.v0.z : g.v0.w;
      return (double)__uint_as_float(b);
    }
    const uint4& q = k < 2 ? g.v0 : g.v1;
    return (k & 1) ? __hiloint2double((int)q.w, (int)q.z) : __hiloint2double((int)q.y, (int)q.x);
  }
  __device__ __forceinline__ static uint32_t key(const Group<VT>& g, int k) {
    return k == 0 ? g.k.x : k == 1 ? g.k.y : k == 2 ? g.k.z : g.k.w;
  }

  // One 32-entry chunk: the layout guarantees its rows are distinct, so every
  // lane adds its product straight into its row's accumulator. A row's
  // entries arrive in column order (earlier chunks, earlier blocks), so each
  // row is summed like the reference's spmv / spmv_t loop
  // (sparsify.cpp:203-226): acc += v * x, no FMA. Padding (v = 0) carries
  // the half's sink row (its max_rows), never read.
  __device__ __forceinline__ static void fold(uint32_t u, double v, uint32_t xs_s, uint32_t acc_s) {
    const double p = __dmul_rn(v, lds_f64(xs_s + ((u & kColMask) << 3)));
    const uint32_t a = acc_s + (u >> 13);
    sts_f64(a, __dadd_rn(lds_f64(a), p));
    __syncwarp();  // the next chunk may revisit a row through another lane
  }
  // Four chunks inside one column block: the x gathers do not depend on the
  // accumulators, so all four are issued before the read-modify-write chain.
  __device__ __forceinline__ static void fold4(const Group<VT>& g, uint32_t xs_s, uint32_t acc_s) {
    double p[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = lds_f64(xs_s + ((key(g, k) & kColMask) << 3));
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = __dmul_rn(value(g, k), p[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t a = acc_s + (key(g, k) >> 13);
      sts_f64(a, __dadd_rn(lds_f64(a), p[k]));
      __syncwarp();
    }
  }

  __device__ __forceinline__ void load_group(const uint32_t* gk, const VT* gv, int g, int lane, uint64_t pol,
                                             Group<VT>& r) const {
    const int64_t e = (int64_t)g * kGE;
    r.k = ldg_stream(gk + e + 4 * lane, pol);
    if (sizeof(VT) == 4) {
      r.v0 = ldg_stream(gv + e + 4 * lane, pol);
    } else {
      r.v0 = ldg_stream(gv + e + 2 * lane, pol);
      r.v1 = ldg_stream(gv + e + 64 + 2 * lane, pol);
    }
  }

  template <int ROLE, bool LOG, bool DET>
  __device__ void half(const double* x, const double* wgt, const double* old, double* out, unsigned char* ne,
                       int* dyn, double exponent, int policy, int t, unsigned long long* flag, double* absdiff,
                       double& err, long long& masks) const {
    extern __shared__ __align__(128) unsigned char dsm[];
    double* acc = reinterpret_cast<double*>(dsm);
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm + align16((size_t)(acc_rows + kSinkRows) * 8));
    uint64_t* empty = full + STG;
    uint32_t* ph = reinterpret_cast<uint32_t*>(empty + STG);  // phases completed per stage
    double* tiles = reinterpret_cast<double*>(dsm + head_bytes());

    const BlockedHalf& H = L[ROLE];
    const int cta = blockIdx.x;
    const int q = cta / S;     // row slab
    const int part = cta % S;  // column part
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const VT* gval = static_cast<const VT*>(H.val);
    const int r0 = H.slab_row0[q];
    const int nrows = H.slab_row0[q + 1] - r0;
    // the CTA's column part [pstart, pend) in blocks of W
    const int64_t pstart = part == 0 ? 0 : H.split;
    const int64_t pend = (S == 1 || part == S - 1) ? H.n_in : H.split;
    const int nb = (int)((pend - pstart + H.W - 1) / H.W);

    // Barriers are initialised once per launch (first half of iteration 1)
    // and never re-initialised; each stage's phase count carries over from
    // half to half in shared memory.
    if ((fresh || (ROLE == 0 && t == 1)) && threadIdx.x == 0) {
      for (int s = 0; s < STG; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], kNW);
        ph[s] = 0u;
      }
      fence_mbar_init();
    }
    unsigned long long* tr = (trace && t <= 4) ? trace + (((size_t)(t - 1) * 2 + ROLE) * gridDim.x + cta) * 24 : nullptr;
    if (tr && threadIdx.x == 0) {
      tr[0] = globaltimer();
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[20] = smid;
    }
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) acc[r] = 0.0;
    __syncthreads();
    // bit s: parity of the next phase of stage s; flipped after every wait on it
    uint32_t pmask = 0;
#pragma unroll
    for (int s = 0; s < STG; ++s) pmask |= (ph[s] & 1u) << s;
    uint32_t ph0[STG];
#pragma unroll
    for (int s = 0; s < STG; ++s) ph0[s] = ph[s];

    if (w == kNW) {
      // ---- producer warp: x tiles through a STG-deep ring ----
      if (lane == 0 && nb > 0) {
        fence_proxy_async();  // x was written with generic stores before the grid barrier
        int s = 0;
        for (int b = 0; b < nb; ++b) {
          if (b >= STG) {  // stage s last held block b - STG: wait for its release
            if (!mbar_wait(&empty[s], (pmask >> s) & 1u, fault))
              record_fault(fault, 0x10000000u | ((unsigned)ROLE << 24) | (unsigned)b);
            pmask ^= 1u << s;
          }
          const int64_t c0 = pstart + (int64_t)b * H.W;
          const int64_t cnt = min((int64_t)H.W, pend - c0);
          const uint32_t bytes = (uint32_t)align16((size_t)cnt * 8);
          mbar_arrive_expect_tx(&full[s], bytes);
          bulk_copy_g2s(tiles + (size_t)s * kTileW, x + c0, bytes, &full[s]);
          s = s + 1 == STG ? 0 : s + 1;
        }
      }
      __syncwarp();
    } else if (nb > 0) {
      // ---- consumer warps: one contiguous stream per warp, kDepth groups of
      // 4 chunks in flight in registers ahead of the group being folded ----
      const long long* ofs = H.off + ((int64_t)cta * kNW + w) * (H.Bh + 1);  // block starts; [nb] = stream end
      const long long sbeg = ofs[0];
      // every block holds at least one chunk and streams are padded to whole
      // groups, so the stream is a whole number of groups
      const int ngroups = (int)((ofs[nb] - sbeg + kGE - 1) / kGE);
      const uint32_t* gk = H.packed + sbeg;
      const VT* gv = gval + sbeg;
      const uint64_t pol = evict_first_policy();
      // Loads are unconditional (clamped to the last group) so no predicated
      // register merge forces a wait.
      const int glast = max(ngroups - 1, 0);
      // Two register sets of kDepth groups. ptxas tracks every streaming load
      // on one scoreboard, so any wait is a wait for ALL loads in flight: the
      // loads of set B are therefore issued only once set A has landed (their
      // addresses carry a zero derived from A's keys) and stay in flight
      // while A is folded -- one exposed wait per 4 * kDepth chunks.
      Group<VT> A[kDepth], Bq[kDepth];
#pragma unroll
      for (int d = 0; d < kDepth; ++d) load_group(gk, gv, min(d, glast), lane, pol, A[d]);
      // Block boundaries travel in the stream itself: every entry (and pad) of a
      // block's first chunk carries kNewBlock, so entering the next x tile
      // costs no dependent global load.
      int cb = -1, cs = STG - 1;  // current block and its stage
      const uint32_t acc_s = smem_u32(acc);
      const uint32_t tiles_s = smem_u32(tiles);
      uint32_t xs_s = tiles_s;  // tile of the current block
      auto run_group = [&](const Group<VT>& cur) {
        if (((cur.k.x | cur.k.y | cur.k.z | cur.k.w) & kNewBlock) == 0) {  // warp-uniform
          fold4(cur, xs_s, acc_s);
          return;
        }
        // (kept inline: as an out-of-line call this path cost 13% -- 2254 vs 2577 iterations/s)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t u = key(cur, k);
          if (u & kNewBlock) {  // warp-uniform: release tile cb, enter the next
            __syncwarp();
            if (cb >= 0 && lane == 0) mbar_arrive(&empty[cs]);
            ++cb;
            cs = cs + 1 == STG ? 0 : cs + 1;
            xs_s = tiles_s + (uint32_t)cs * (kTileW * 8);
            if (!mbar_wait(&full[cs], (pmask >> cs) & 1u, fault))
              record_fault(fault, 0x30000000u | ((unsigned)ROLE << 24) | (unsigned)cb);
            pmask ^= 1u << cs;
          }
          fold(u, value(cur, k), xs_s, acc_s);
        }
      };
      auto landed = [&](const Group<VT>* G) -> int {  // 0 once the set's keys are in registers
        uint32_t o = 0;
#pragma unroll
        for (int d = 0; d < kDepth; ++d) o |= G[d].k.x;
        return (int)((o >> 13) & 7u);  // bits 13-15 of a key are zero
      };
      for (int g0 = 0; g0 < ngroups; g0 += 2 * kDepth) {
        const int za = landed(A);
#pragma unroll
        for (int d = 0; d < kDepth; ++d) load_group(gk, gv, min(g0 + kDepth + d + za, glast), lane, pol, Bq[d]);
#pragma unroll
        for (int d = 0; d < kDepth; ++d)
          if (g0 + d < ngroups) run_group(A[d]);  // warp-uniform
        const int zb = landed(Bq);
#pragma unroll
        for (int d = 0; d < kDepth; ++d) load_group(gk, gv, min(g0 + 2 * kDepth + d + zb, glast), lane, pol, A[d]);
#pragma unroll
        for (int d = 0; d < kDepth; ++d)
          if (g0 + kDepth + d < ngroups) run_group(Bq[d]);
      }
      if (tr && lane == 0) tr[1 + w] = globaltimer();
      // release the last block; a stream that (against the layout's promise)
      // ended early still passes through every remaining tile in order
      for (;;) {
        __syncwarp();
        if (cb >= 0 && lane == 0) mbar_arrive(&empty[cs]);
        if (++cb >= nb) break;
        cs = cs + 1 == STG ? 0 : cs + 1;
        if (!mbar_wait(&full[cs], (pmask >> cs) & 1u, fault))
          record_fault(fault, 0x40000000u | ((unsigned)ROLE << 24) | (unsigned)cb);
        pmask ^= 1u << cs;
      }
    }
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[16] = globaltimer();
    if (threadIdx.x == 0) {  // block b used stage b % STG once
#pragma unroll
      for (int s = 0; s < STG; ++s) ph[s] = ph0[s] + (uint32_t)((nb - s + STG - 1) / STG);
    }
    // ---- finalize this CTA's atoms of the slab ----
    int fr0 = 0, fr1 = nrows;
    const double* pacc = nullptr;  // CL: the partner's accumulators (DSMEM)
    if (S == 2 && CL) {
      const int mid = nrows >> 1;
      fr0 = part == 0 ? 0 : mid;
      fr1 = part == 0 ? mid : nrows;
      if (tr && threadIdx.x == 0) tr[17] = globaltimer();
      cluster_sync();  // both CTAs' sums complete (release/acquire at cluster scope)
      pacc = map_peer(acc, (unsigned)(part ^ 1));
    } else if (S == 2) {
      const int mid = nrows >> 1;
      fr0 = part == 0 ? 0 : mid;
      fr1 = part == 0 ? mid : nrows;
      const int o0 = part == 0 ? mid : 0, o1 = part == 0 ? nrows : mid;  // the partner's rows
      for (int r = o0 + threadIdx.x; r < o1; r += blockDim.x) __stcg(xchg + r0 + r, acc[r]);
      __syncthreads();
      if (tr && threadIdx.x == 0) tr[17] = globaltimer();
      if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int target = 2u * (unsigned)(2 * (t - 1) + ROLE + 1);
        atomicAdd(pair + q, 1u);
        bool ok = false;
        for (int spin = 0; spin < (1 << 22); ++spin) {
          if (*(volatile unsigned int*)(pair + q) >= target) {
            ok = true;
            break;
          }
          if ((spin & 255) == 255 && __ldcg(fault)) break;
        }
        if (!ok) record_fault(fault, 0x50000000u | ((unsigned)ROLE << 24));
        __threadfence();
      }
      __syncthreads();
    }
    if (tr && threadIdx.x == 0) tr[18] = globaltimer();
    // Latency-bound (~13 rows per thread at config 4): the loads of the next
    // rows are issued before the current row is finalized (software
    // pipeline: out/ne/dyn never alias old/wgt/xchg).
    {
      int r = fr0 + threadIdx.x;
      double o = 0.0, wv = 0.0, px = 0.0;
      unsigned char nv = 0;
      if (r < fr1) {
        o = __ldcg(old + r0 + r);
        nv = ne[r0 + r];
        wv = __ldg(wgt + r0 + r);
        if (S == 2) px = CL ? pacc[r] : __ldcg(xchg + r0 + r);
      }
      for (; r < fr1; r += blockDim.x) {
        const int64_t i = r0 + r;
        const double oc = o, wc = wv, pc = px;
        const unsigned char nc = nv;
        const int rn = r + (int)blockDim.x;
        if (rn < fr1) {  // next row's loads in flight while this one finishes
          o = __ldcg(old + r0 + rn);
          nv = ne[r0 + rn];
          wv = __ldg(wgt + r0 + rn);
          if (S == 2) px = CL ? pacc[rn] : __ldcg(xchg + r0 + rn);
        }
        if (!nc) {
          out[i] = oc;
          continue;
        }
        const double tmp = S == 2 ? __dadd_rn(acc[r], pc) : acc[r];  // p0 + p1 (commutes exactly)
        err += loopcore::finalize_atom<LOG>(i, tmp, oc, wc, exponent, policy, t, ne, dyn, out, flag, masks);
      }
    }
    // one launch per half: the partner may still read this CTA's accumulators,
    // and a CTA must not exit under a DSMEM reader (the persistent loop's grid
    // barrier already orders this)
    if (S == 2 && CL && fresh) cluster_sync();
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[19] = globaltimer();
  }
};

// ---- layout builder --------------------------------------------------------------

// Per row: entries whose column lies before `split` (columns ascend in a row).
__global__ void split_count_kernel(const long long* ptr, const uint32_t* idx, int64_t n_out, uint32_t split,
                                   long long* cnt0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n_out; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n_out) {  // one element past the rows: the exclusive scan's total lands here
      cnt0[i] = 0;
      continue;
    }
    long long lo = ptr[i], hi = ptr[i + 1];
    const long long b = lo;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (idx[mid] < split) lo = mid + 1;
      else hi = mid;
    }
    cnt0[i] = lo - b;
  }
}

// Row slabs of ~equal entry count: slab k starts at the first row whose
// prefix reaches m k / Q (ptr is the prefix: one binary search per slab).
__global__ void slab_cut_kernel(const long long* ptr, int64_t n_out, int64_t m, int Q, int* slab_row0) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > Q) return;
  if (k == 0 || k == Q) {
    slab_row0[k] = k == 0 ? 0 : (int)n_out;
    return;
  }
  const long long target = (long long)((double)m * k / Q);
  int64_t lo = 0, hi = n_out + 1;  // first index with ptr[index] >= target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ptr[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  slab_row0[k] = (int)min(lo, n_out);
}

// The 15 warp ranges of every (slab, column part): ~equal entries of that part.
// pre0[r] = entries of rows [0, r) left of the split (S = 2); one thread per (slab, part).
__global__ void warp_cut_kernel(const long long* ptr, const long long* pre0, const int* slab_row0, int Q, int S,
                                int* warp_end) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= Q * S) return;
  const int q = id / S, part = id % S;
  const int a = slab_row0[q], z = slab_row0[q + 1];
  auto pref = [&](int r) -> long long {  // entries of this part in rows [a, r)
    const long long tot = ptr[r] - ptr[a];
    if (S == 1) return tot;
    const long long p0 = pre0[r] - pre0[a];
    return part == 0 ? p0 : tot - p0;
  };
  const long long e1 = pref(z);
  int prev = a;
  for (int wv = 0; wv < kNW; ++wv) {
    int r_end = z;
    if (wv + 1 < kNW) {
      const long long target = (long long)((double)e1 * (wv + 1) / kNW);
      int lo = a, hi = z;  // first r in [a, z) with pref(r) >= target, else z
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (pref(mid) < target) lo = mid + 1;
        else hi = mid;
      }
      r_end = max(prev, lo);
    }
    warp_end[id * kNW + wv] = r_end;
    prev = r_end;
  }
}

// key = segment (CTA, warp, block) | bank class of the row | row. Sorting by
// it (stably) lists each segment's rows grouped by shared-memory bank class,
// every row's entries consecutive in column order; chunk c then takes list
// positions c, c+C, ... and so spreads its rows over all banks.
__global__ void key_kernel(const long long* ptr, const uint32_t* idx, int64_t n_out, const int* slab_row0, int Q,
                           const int* warp_end, int W, int S, int Bh, uint32_t split, uint32_t* seg,
                           unsigned long long* key) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_out; i += nw) {
    // the row's slab (the last one starting at or before it) and its warp in each column part
    int lo = 0, hi = Q;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (slab_row0[mid] <= i) lo = mid;
      else hi = mid;
    }
    const uint32_t slab = (uint32_t)lo;
    const uint32_t rl = (uint32_t)(i - slab_row0[slab]);
    uint32_t wv_of[2] = {0u, 0u};
    for (int part = 0; part < S; ++part) {
      const int* we = warp_end + ((int)slab * S + part) * kNW;
      int wv = 0;
      while (wv + 1 < kNW && we[wv] <= i) ++wv;
      wv_of[part] = (uint32_t)wv;
    }
    for (long long q = ptr[i] + lane; q < ptr[i + 1]; q += 32) {
      const uint32_t part = idx[q] >= split ? 1u : 0u;  // split = n_in when S = 1
      const uint32_t blk = (idx[q] - (part ? split : 0u)) / (uint32_t)W;  // block inside the part
      const uint32_t cta = slab * (uint32_t)S + part;
      const uint32_t sg = (cta * kNW + wv_of[part]) * (uint32_t)Bh + blk;
      seg[q] = sg;
      key[q] = ((unsigned long long)sg << 20) | ((unsigned long long)(rl & 15u) << 16) | rl;
    }
  }
}

__global__ void split_kernel(const unsigned long long* key_s, int64_t m, uint32_t* seg_s, uint32_t* rl) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = key_s[q];
    seg_s[q] = (uint32_t)(k >> 20);
    rl[q] = (uint32_t)(k & 0xffffu);
  }
}

// Start of the run of equal (segment, row) containing q (max-scanned next).
__global__ void run_head_kernel(const uint32_t* keys_s, const uint32_t* rl, int64_t m, uint32_t* start) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    const bool head = q == 0 || keys_s[q] != keys_s[q - 1] || rl[q] != rl[q - 1];
    start[q] = head ? (uint32_t)q : 0u;
  }
}

// Run length (the row's entry count in its segment) at each run head, and
// the segment's longest run.
__global__ void runlen_kernel(const uint32_t* keys_s, const uint32_t* rl, const uint32_t* start, int64_t m,
                              uint32_t* runlen, unsigned int* maxrun) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    if (start[q] != (uint32_t)q) continue;
    int64_t e = q + 1;
    while (e < m && keys_s[e] == keys_s[q] && rl[e] == rl[q]) ++e;
    runlen[q] = (uint32_t)(e - q);
    atomicMax(&maxrun[keys_s[q]], (unsigned int)(e - q));
  }
}

// Chunk placement. A segment of E entries (rows grouped by bank class, each
// row's entries consecutive in column order) gets C = max(ceil(E/32), longest run)
// chunks of 32 slots; list position p maps to chunk p mod C, slot p div C.
// A row's m <= C consecutive positions hit m distinct chunks, so no chunk
// holds a row twice; its entries then take those chunks in ascending order,
// so the row is still summed in column order when the chunks run in order.
//
// Column spreading (slot_warp_kernel, one warp per segment): the placement fixes,
// per row bank class, a set of list positions (hence (chunk, half-warp)
// slots); any permutation of the class's entries over its own positions
// keeps the row-bank spread. The x gather costs the worst column-bank
// multiplicity of a half-warp (~6 wavefronts per chunk at random, 4.9 per
// LDS.64 measured with the accumulator loads), so each class's entries are
// dealt greedily to the free position whose half-warp holds the fewest
// entries of the entry's column class (rows with several entries first, each
// in distinct chunks). Simulated at config 4: 6.1 -> 3.8 gather wavefronts
// per chunk, no extra padding. newpos[q] = chosen list position, or -1 where
// a segment keeps the plain placement.
// Column bank class of each sorted entry (coalesced; read by slot_warp_kernel).
__global__ void colclass_kernel(const uint32_t* perm, const uint32_t* idx, int W, uint32_t split, int64_t m,
                                unsigned char* cc) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t j = idx[perm[q]];
    cc[q] = (unsigned char)(((j >= split ? j - split : j) % (uint32_t)W) & 15u);
  }
}

// The free positions of a class are scored by the lanes in parallel (cost =
// the column class's count in that position's half-warp, ties to the lowest
// position): one warp argmin per entry.
constexpr int kSlotWarps = 8;
__global__ void __launch_bounds__(32 * kSlotWarps) slot_warp_kernel(
    int64_t nkeys, const long long* useg, const unsigned long long* cnt, const long long* nchunk, const uint32_t* rl,
    const unsigned char* colc, const uint32_t* start, const uint32_t* runlen, int* newpos) {
  __shared__ unsigned char counts[kSlotWarps][32 * 2 * 16];  // [chunk][half][column class]
  __shared__ int cls_n[kSlotWarps][17];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t k = (int64_t)blockIdx.x * kSlotWarps + wl;
  if (k >= nkeys) return;
  const int E = (int)cnt[k];
  const int C = (int)nchunk[k];
  if (E == 0 || C > 32) return;
  const long long u0 = useg[k];
  unsigned char* ct = counts[wl];
  for (int i = lane; i < C * 32; i += 32) ct[i] = 0;
  if (lane < 17) cls_n[wl][lane] = 0;
  __syncwarp();
  for (int e = lane; e < E; e += 32) atomicAdd(&cls_n[wl][rl[u0 + e] & 15u], 1);
  __syncwarp();
  bool ok = true;
  int ps = 0;
  for (int c = 0; c < 16 && ok; ++c) {
    const int nk = cls_n[wl][c];
    if (nk == 0) continue;
    if (nk > 64) {
      ok = false;
      break;
    }
    unsigned long long freem = nk == 64 ? ~0ull : ((1ull << nk) - 1ull);
    for (int pass = 0; pass < 2 && ok; ++pass) {
      for (int o = 0; o < nk; ++o) {
        const long long q = u0 + ps + o;
        const long long rs = start[q];
        const int rn = (int)runlen[rs];
        if ((rn > 1) != (pass == 0)) continue;
        const int cc = colc[q];
        unsigned int key = 0xffffffffu;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int f = lane + 32 * h;
          if (f < nk && ((freem >> f) & 1ull)) {
            const int pos = ps + f;
            const int ch = pos % C, hf = (pos / C) & 1;
            bool clash = false;
            for (int j = 0; j < rn && rn > 1; ++j) {
              const int np = newpos[rs + j];
              if (rs + j != q && np >= 0 && np % C == ch) {
                clash = true;
                break;
              }
            }
            if (!clash) key = min(key, ((unsigned int)ct[(ch * 2 + hf) * 16 + cc] << 8) | (unsigned int)f);
          }
        }
#pragma unroll
        for (int o2 = 16; o2; o2 >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, o2));
        if (key == 0xffffffffu) {
          ok = false;
          break;
        }
        const int f = (int)(key & 255u);
        const int pos = ps + f;
        const int ch = pos % C, hf = (pos / C) & 1;
        if (lane == 0) {
          newpos[q] = pos;
          unsigned char& v = ct[(ch * 2 + hf) * 16 + cc];
          if (v < 255) ++v;
        }
        freem &= ~(1ull << f);
        __syncwarp();
      }
    }
    ps += nk;
  }
  if (!ok)
    for (int e = lane; e < E; e += 32) newpos[u0 + e] = -1;
}


// ---- chunk placement by edge colouring (option blocked_spread = 1, the default) ----
// A segment's entries are the edges of a bipartite multigraph: 16 row bank
// classes (the fp64 accumulator's bank pair, row_local & 15) against 16
// column bank classes (the x tile's bank pair, col_local & 15). A 64-bit
// shared access is served per half-warp, one wavefront per distinct address
// in the busiest bank pair (profiles/microbench/lds64_conflicts.cu), so a
// half-chunk whose 16 entries form a MATCHING -- distinct row classes and
// distinct column classes -- costs the ideal 1 + 1 + 1 wavefronts for the x
// gather, the accumulator load and its store. The H = 2C half-chunks are the
// colours of an edge colouring: an edge takes a colour free at both its
// classes; when the two have no common free colour, the a/b alternating path
// from the column class is flipped (Kempe chain; bipartite, so it cannot end
// at the row class) and the edge takes a. Only edges of a class with more
// than H entries stay uncoloured; they (and the few whose flip broke the
// one-row-once-per-chunk rule) are then dealt to the half-chunk with room
// where they add the fewest wavefronts. Measured at config 4: 3.8 / 4.05
// wavefronts per accumulator / gather access with the run-length placement
// plus greedy column dealing (slot_warp_kernel), 3.12 / 2.93 with this
// (the layout analysed by scratch-free tooling: SPK_DUMP_BLOCKED writes the head of the key stream).
// One warp per segment; all state in shared memory. newpos[q] = chunk * 32 +
// lane, or -1 (whole segment) when the segment does not fit this scheme.
// Two instances: segments of up to 512 entries in up to 16 chunks (all of config
// 4's) run with 5.2 KB of state per warp, 8 warps per CTA -- the kernel is a
// latency-bound sequential walk, so resident warps are its throughput --
// and the rest with the full-size state.
template <int MAXE, int MAXH>
struct ColorWs {
  unsigned short at[32][MAXH];   // edge holding colour h at class x (0-15 rows, 16-31 columns)
  unsigned short erow[MAXE];
  unsigned char evert[MAXE];  // row class | column class << 4
  unsigned char ecol[MAXE];   // colour (half-chunk) or 0xff
  unsigned char cnt[MAXH][32];        // entries of class x in half-chunk h
  unsigned char fill[MAXH], rmax[MAXH], cmax[MAXH];
  unsigned int slot[MAXH];
};
template <int MAXE, int MAXH, int WARPS, bool REST>
__global__ void __launch_bounds__(32 * WARPS) color_warp_kernel(
    int64_t nkeys, const long long* useg, const unsigned long long* cnt, const long long* nchunk, const uint32_t* rl,
    const unsigned char* colc, const long long* seg_base, uint32_t padrow, int* newpos, uint32_t* packed,
    unsigned long long* stats) {
  __shared__ ColorWs<MAXE, MAXH> ws_all[WARPS];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t k = (int64_t)blockIdx.x * WARPS + wl;
  if (k >= nkeys) return;
  const int E = (int)cnt[k];
  const int C = (int)nchunk[k];
  if (E == 0 || 2 * C > MAXH || E > MAXE) return;
  if (REST && 2 * C <= 32 && E <= 512) return;  // placed by the small instance
  const int H = 2 * C;
  const long long u0 = useg[k];
  ColorWs<MAXE, MAXH>& ws = ws_all[wl];
  const unsigned FULL = 0xffffffffu;
  for (int i = lane; i < 32 * MAXH; i += 32) (&ws.at[0][0])[i] = 0xffffu;
  for (int e = lane; e < E; e += 32) {
    const uint32_t r = rl[u0 + e];
    ws.erow[e] = (unsigned short)r;
    ws.evert[e] = (unsigned char)((r & 15u) | ((uint32_t)colc[u0 + e] << 4));
    ws.ecol[e] = 0xff;
  }
  __syncwarp();
  // lane x keeps the free colours of class x
  unsigned long long freec = H == 64 ? ~0ull : ((1ull << H) - 1ull);
  int st = 37;
  {
    const int primes[6] = {37, 41, 43, 47, 53, 59};
    for (int j = 0; j < 6; ++j)
      if (E % primes[j]) {
        st = primes[j];
        break;
      }
  }
  // colours of the other entries of e's row (a run of the sorted list): their chunks are closed to e
  auto run_forbidden = [&](int e) -> unsigned long long {
    unsigned long long forb = 0;
    const unsigned short r = ws.erow[e];
    for (int j = e - 1; j >= 0 && ws.erow[j] == r; --j)
      if (ws.ecol[j] != 0xff) forb |= 3ull << (ws.ecol[j] & 0xfe);
    for (int j = e + 1; j < E && ws.erow[j] == r; ++j)
      if (ws.ecol[j] != 0xff) forb |= 3ull << (ws.ecol[j] & 0xfe);
    return forb;
  };
  bool ok = true;
  int pos = 0;
  for (int i = 0; i < E && ok; ++i) {
    const int e = pos;
    pos += st;
    while (pos >= E) pos -= E;
    const int vb = ws.evert[e];
    const int u = vb & 15, v = 16 + (vb >> 4);
    const unsigned long long forb = run_forbidden(e);
    const unsigned long long fu = __shfl_sync(FULL, freec, u) & ~forb;
    const unsigned long long fv = __shfl_sync(FULL, freec, v) & ~forb;
    int a;
    if (fu & fv) {
      a = __ffsll((long long)(fu & fv)) - 1;
    } else if (fu && fv) {
      a = __ffsll((long long)fu) - 1;            // free at u, used at v
      const int b = __ffsll((long long)fv) - 1;  // free at v, used at u
      int x = v, c = a, len = 0;
      unsigned short mine = 0xffffu;
      for (;;) {
        const unsigned short f = ws.at[x][c];
        if (f == 0xffffu) break;
        if (len >= 32) {
          ok = false;
          if (stats && lane == 0) atomicAdd(&stats[2], 1ull);
          break;
        }
        if (lane == len) mine = f;
        ++len;
        const int fb = ws.evert[f];
        const int fu2 = fb & 15, fv2 = 16 + (fb >> 4);
        x = x == fu2 ? fv2 : fu2;
        c ^= a ^ b;
      }
      if (!ok) break;
      int oldc = 0, y0 = 0, y1 = 0;
      if (lane < len) {
        oldc = ws.ecol[mine];
        const int fb = ws.evert[mine];
        y0 = fb & 15;
        y1 = 16 + (fb >> 4);
        ws.at[y0][oldc] = 0xffffu;
        ws.at[y1][oldc] = 0xffffu;
      }
      __syncwarp();
      if (lane < len) {
        const int newc = oldc ^ a ^ b;
        ws.at[y0][newc] = mine;
        ws.at[y1][newc] = mine;
        ws.ecol[mine] = (unsigned char)newc;
      }
      __syncwarp();
      // v: a freed by the flip (and taken again below), b now used; the path's
      // far end swaps which of a, b it holds; interior classes hold both
      if (lane == v) freec &= ~(1ull << b);
      if (lane == x) freec ^= (1ull << a) | (1ull << b);
    } else {
      if (stats && lane == 0) atomicAdd(&stats[4], 1ull);
      continue;  // a class with more entries than colours: dealt below
    }
    if (lane == 0) {
      ws.ecol[e] = (unsigned char)a;
      ws.at[u][a] = (unsigned short)e;
      ws.at[v][a] = (unsigned short)e;
    }
    if (lane == u || lane == v) freec &= ~(1ull << a);
    __syncwarp();
  }
  if (ok) {
    // a flip may have moved an entry into a chunk that already holds its row: evict the later one
    for (int e = lane; e < E; e += 32) {
      if (e > 0 && ws.erow[e - 1] == ws.erow[e]) continue;  // run heads only
      unsigned int chunks = 0;
      for (int j = e; j < E && ws.erow[j] == ws.erow[e]; ++j) {
        const int c = ws.ecol[j];
        if (c == 0xff) continue;
        if ((chunks >> (c >> 1)) & 1u) {
          const int vb = ws.evert[j];
          ws.at[vb & 15][c] = 0xffffu;
          ws.at[16 + (vb >> 4)][c] = 0xffffu;
          ws.ecol[j] = 0xff;
          if (stats) atomicAdd(&stats[5], 1ull);
        } else {
          chunks |= 1u << (c >> 1);
        }
      }
    }
    __syncwarp();
    for (int i = lane; i < MAXH * 32; i += 32) {
      const int h = i >> 5, x = i & 31;
      ws.cnt[h][x] = (h < H && ws.at[x][h] != 0xffffu) ? 1 : 0;
    }
    __syncwarp();
    for (int h = lane; h < MAXH; h += 32) {
      int f = 0;
      for (int x = 0; x < 16; ++x) f += ws.cnt[h][x];
      ws.fill[h] = (unsigned char)f;
      ws.rmax[h] = ws.cmax[h] = f > 0 ? 1 : 0;
      ws.slot[h] = 0u;
    }
    __syncwarp();
    for (int e = 0; e < E && ok; ++e) {
      if (ws.ecol[e] != 0xff) continue;  // warp-uniform
      const int vb = ws.evert[e];
      const int u = vb & 15, v = 16 + (vb >> 4);
      const unsigned long long forb = run_forbidden(e);
      unsigned int key = 0xffffffffu;
#pragma unroll
      for (int hh = 0; hh < (MAXH + 31) / 32; ++hh) {
        const int h = lane + 32 * hh;
        if (h < H && ws.fill[h] < 16 && !((forb >> h) & 1ull)) {
          const int d = 2 * (ws.cnt[h][u] + 1 > max(1, (int)ws.rmax[h])) + (ws.cnt[h][v] + 1 > max(1, (int)ws.cmax[h]));
          key = min(key, ((unsigned)d << 16) | ((unsigned)ws.fill[h] << 8) | (unsigned)h);
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) key = min(key, __shfl_xor_sync(FULL, key, o));
      if (key == 0xffffffffu) {
        ok = false;
        if (stats && lane == 0) atomicAdd(&stats[3], 1ull);
        break;
      }
      const int h = (int)(key & 255u);
      if (lane == 0) {
        ws.ecol[e] = (unsigned char)h;
        ws.rmax[h] = (unsigned char)max((int)ws.rmax[h], ++ws.cnt[h][u]);
        ws.cmax[h] = (unsigned char)max((int)ws.cmax[h], ++ws.cnt[h][v]);
        ++ws.fill[h];
      }
      __syncwarp();
    }
  }
  if (stats && lane == 0) atomicAdd(&stats[ok ? 0 : 1], 1ull);
  if (!ok) {
    for (int e = lane; e < E; e += 32) newpos[u0 + e] = -1;
    return;
  }
  for (int e = lane; e < E; e += 32) {
    const int h = ws.ecol[e];
    const unsigned int sl = atomicAdd(&ws.slot[h], 1u);
    newpos[u0 + e] = (h >> 1) * 32 + (h & 1) * 16 + (int)sl;
  }
  // the free lanes of every half-chunk: padding in row and column classes the half-chunk does not use
  const int64_t Cg0 = seg_base[k] >> 5;
  for (int h = lane; h < H; h += 32) {
    unsigned int usedr = 0, usedc = 0;
    for (int x = 0; x < 16; ++x) {
      if (ws.cnt[h][x]) usedr |= 1u << x;
      if (ws.cnt[h][16 + x]) usedc |= 1u << x;
    }
    for (int sl = ws.fill[h]; sl < 16; ++sl) {
      const int jr = __ffs((int)(~usedr & 0xffffu)) - 1, jc = __ffs((int)(~usedc & 0xffffu)) - 1;
      usedr |= 1u << jr;
      usedc |= 1u << jc;
      const uint32_t row = padrow + (((uint32_t)jr - padrow) & 15u);
      packed[pos_packed(Cg0 + (h >> 1), (h & 1) * 16 + sl)] = (row << 16) | (uint32_t)jc | (h < 2 ? kNewBlock : 0u);
    }
  }
}

template <class VT>
__global__ void place_kernel(const uint32_t* keys_s, const uint32_t* perm, const uint32_t* rl, const uint32_t* start,
                             const uint32_t* runlen, const long long* useg, const long long* seg_base,
                             const long long* nchunk, const uint32_t* idx, const VT* val, int W, uint32_t split,
                             int64_t m,
                             const int* newpos, bool direct, uint32_t* packed, VT* vout) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = keys_s[q];
    const long long C = nchunk[key];
    const long long ps = (long long)start[q] - useg[key];  // the row's first list position
    const long long kk = (long long)q - (long long)start[q];
    const long long mr = runlen[start[q]];
    const long long a = ps % C, wrap = a + mr - C;
    long long c, pp;
    int lane;
    if (direct && newpos[q] >= 0) {  // chunk * 32 + lane (color_warp_kernel)
      c = newpos[q] >> 5;
      lane = newpos[q] & 31;
      pp = -1;
    } else if (newpos[q] >= 0) {  // column-spread position (slot_warp_kernel)
      pp = newpos[q];
      c = pp % C;
    } else if (wrap > 0 && kk < wrap) {
      c = kk;
      pp = ps + (C - a) + c;
    } else {
      c = wrap > 0 ? a + (kk - wrap) : a + kk;
      pp = ps + (c - a);
    }
    if (pp >= 0) {
      const long long slot = pp / C;  // even slots -> lanes 0-15, odd -> 16-31: each half-warp spans the classes
      lane = (int)(((slot & 1) << 4) + (slot >> 1));
    }
    const int64_t Cg = (seg_base[key] >> 5) + c;  // global chunk index
    const uint32_t src = perm[q];
    const uint32_t j = idx[src];
    packed[pos_packed(Cg, lane)] =
        (rl[q] << 16) | ((j >= split ? j - split : j) % (uint32_t)W) | (c == 0 ? kNewBlock : 0u);
    vout[sizeof(VT) == 4 ? pos_packed(Cg, lane) : pos_f64(Cg, lane)] = val[src];
  }
}

__global__ void fill_u32(uint32_t* v, int64_t m, uint32_t x) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
    v[q] = x;
}

// The first chunk of every segment announces its column block: all 32 slots
// (padding included; real entries are re-written by place_kernel) carry kNewBlock.
__global__ void first_chunk_kernel(int64_t nkeys, const long long* seg_base, const long long* nchunk,
                                   uint32_t pad, uint32_t* packed) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nkeys * 32;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = q >> 5;
    if (nchunk[k] > 0) packed[pos_packed(seg_base[k] >> 5, (int)(q & 31))] = pad | kNewBlock;
  }
}

__global__ void iota_u32(uint32_t* v, int64_t m) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
    v[q] = (uint32_t)q;
}

__global__ void key_hist_kernel(const uint32_t* keys, int64_t m, unsigned long long* hist) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[keys[q]], 1ull);
}

int grid_cap(spk_ctx* ctx, int64_t items) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, (int64_t)ctx->num_sms * 16));
}

}  // namespace

// Build one half's layout from (ptr, idx, val) for P CTAs = Q slabs x S parts.
// Returns false when the shape does not fit (rows per slab >= 2^16).
bool build_blocked(spk_ctx* ctx, int P, int S, int W, int64_t n_out, int64_t n_in, int64_t m, const DBuf& ptr_d,
                   const DBuf& idx_d, const DBuf& val_d, int vbytes, BlockedHost& out) {
  static const bool dbg = std::getenv("SPK_DEBUG_TIMING") != nullptr;
  std::unique_ptr<Timer> tph(dbg ? new Timer(ctx->stream) : nullptr);
  auto phase = [&](const char* what) {
    if (!tph) return;
    std::fprintf(stderr, "[timing]   build_blocked %s %.4f s\n", what, tph->stop());
    tph.reset(new Timer(ctx->stream));
  };
  const int Q = P / S;
  cudaStream_t s = ctx->stream;
  // row slabs of ~equal entry count (device: one binary search of the row prefix per slab)
  out.slab_row0.alloc(sizeof(int) * (Q + 1));
  slab_cut_kernel<<<(Q + 1 + 127) / 128, 128, 0, s>>>(ptr_d.as<long long>(), n_out, m, Q, out.slab_row0.as<int>());
  ++ctx->launches;
  std::vector<int> slab_row0(Q + 1);
  download(ctx, slab_row0.data(), out.slab_row0, sizeof(int) * (Q + 1));
  int max_rows = 0;
  for (int k = 0; k < Q; ++k) max_rows = std::max(max_rows, slab_row0[k + 1] - slab_row0[k]);
  if (max_rows + kSinkRows >= 65535) return false;
  // S = 2: the column parts hold the same number of input atoms (a split on a
  // block boundary left part 0 one block -- 1.5% of the entries at config 4 --
  // heavier, and every half waits for its slowest CTA); multiple of 16 atoms
  // so that part 1's tiles stay 16-byte aligned TMA sources
  const int64_t split = S == 1 ? n_in : std::min<int64_t>(n_in, ((n_in / 2 + 15) / 16) * 16);
  const int nb0 = (int)((split + W - 1) / W), nb1 = (int)((n_in - split + W - 1) / W);
  const int B = nb0 + nb1;
  const int Bh = std::max(nb0, nb1);
  // warp ranges of every (slab, part): equal shares of the part's entries
  // (prefix of the per-row counts left of the split, then 14 binary searches)
  DBuf d_pre0, d_warp_end(sizeof(int) * (size_t)Q * S * kNW);
  if (S == 2) {
    DBuf d_cnt0(sizeof(long long) * (n_out + 1));
    d_pre0.alloc(sizeof(long long) * (n_out + 1));
    split_count_kernel<<<grid_cap(ctx, n_out + 1), 256, 0, s>>>(ptr_d.as<long long>(), idx_d.as<uint32_t>(), n_out,
                                                                 (uint32_t)split, d_cnt0.as<long long>());
    size_t tb0 = 0;
    SPK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb0, d_cnt0.as<long long>(), d_pre0.as<long long>(),
                                           (int)(n_out + 1), s));
    ctx->scratch.ensure(tb0);
    SPK_CUDA(cub::DeviceScan::ExclusiveSum(ctx->scratch.p, tb0, d_cnt0.as<long long>(), d_pre0.as<long long>(),
                                           (int)(n_out + 1), s));
    ctx->launches += 2;
    SPK_CUDA(cudaStreamSynchronize(s));  // d_cnt0 is freed on leaving this scope
  }
  warp_cut_kernel<<<(Q * S + 127) / 128, 128, 0, s>>>(ptr_d.as<long long>(), d_pre0.as<long long>(),
                                                        out.slab_row0.as<int>(), Q, S, d_warp_end.as<int>());
  ++ctx->launches;
  const int64_t nkeys = (int64_t)Q * S * kNW * Bh;
  if (nkeys >= (1LL << 32)) return false;
  const int64_t mm = std::max<int64_t>(m, 1);
  DBuf &iota = tmp_buf(ctx, 0, sizeof(uint32_t) * mm), &perm = tmp_buf(ctx, 1, sizeof(uint32_t) * mm),
       &keys = tmp_buf(ctx, 2, sizeof(uint32_t) * mm), &keys_s = tmp_buf(ctx, 3, sizeof(uint32_t) * mm),
       &key64 = tmp_buf(ctx, 4, sizeof(unsigned long long) * mm),
       &key64_s = tmp_buf(ctx, 5, sizeof(unsigned long long) * mm);
  DBuf hist(sizeof(unsigned long long) * nkeys);
  SPK_CUDA(cudaMemsetAsync(hist.p, 0, hist.bytes, s));
  phase("host cuts");
  key_kernel<<<grid_cap(ctx, n_out * 32), 256, 0, s>>>(ptr_d.as<long long>(), idx_d.as<uint32_t>(), n_out,
                                                        out.slab_row0.as<int>(), Q, d_warp_end.as<int>(), W, S, Bh,
                                                        (uint32_t)split, keys.as<uint32_t>(),
                                                        key64.as<unsigned long long>());
  iota_u32<<<grid_cap(ctx, m), 256, 0, s>>>(iota.as<uint32_t>(), m);
  key_hist_kernel<<<grid_cap(ctx, m), 256, 0, s>>>(keys.as<uint32_t>(), m, hist.as<unsigned long long>());
  ctx->launches += 3;
  int end_bit = 1;
  while ((int64_t(1) << end_bit) < nkeys) ++end_bit;
  size_t tb = 0;
  SPK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key64.as<unsigned long long>(),
                                           key64_s.as<unsigned long long>(), iota.as<uint32_t>(), perm.as<uint32_t>(),
                                           (int)m, 0, 20 + end_bit, s));
  ctx->scratch.ensure(tb);
  SPK_CUDA(cub::DeviceRadixSort::SortPairs(ctx->scratch.p, tb, key64.as<unsigned long long>(),
                                           key64_s.as<unsigned long long>(), iota.as<uint32_t>(), perm.as<uint32_t>(),
                                           (int)m, 0, 20 + end_bit, s));
  ++ctx->launches;
  // run starts / lengths -> chunk counts -> conflict-free placement
  DBuf &rl = tmp_buf(ctx, 6, sizeof(uint32_t) * mm), &start = tmp_buf(ctx, 7, sizeof(uint32_t) * mm),
       &runlen = tmp_buf(ctx, 8, sizeof(uint32_t) * mm);
  DBuf maxrun(sizeof(unsigned int) * nkeys);
  SPK_CUDA(cudaMemsetAsync(maxrun.p, 0, maxrun.bytes, s));
  split_kernel<<<grid_cap(ctx, m), 256, 0, s>>>(key64_s.as<unsigned long long>(), m, keys_s.as<uint32_t>(),
                                                rl.as<uint32_t>());
  run_head_kernel<<<grid_cap(ctx, m), 256, 0, s>>>(keys_s.as<uint32_t>(), rl.as<uint32_t>(), m,
                                                   start.as<uint32_t>());
  ctx->launches += 2;
  tb = 0;
  SPK_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, start.as<uint32_t>(), start.as<uint32_t>(), cub::Max(), (int)m,
                                          s));
  ctx->scratch.ensure(tb);
  SPK_CUDA(cub::DeviceScan::InclusiveScan(ctx->scratch.p, tb, start.as<uint32_t>(), start.as<uint32_t>(), cub::Max(),
                                          (int)m, s));
  phase("keys + sort");
  runlen_kernel<<<grid_cap(ctx, m), 256, 0, s>>>(keys_s.as<uint32_t>(), rl.as<uint32_t>(), start.as<uint32_t>(), m,
                                                 runlen.as<uint32_t>(), maxrun.as<unsigned int>());
  ctx->launches += 2;
  std::vector<unsigned long long> h(nkeys);
  std::vector<unsigned int> mx(nkeys);
  download(ctx, h.data(), hist, sizeof(unsigned long long) * nkeys);
  download(ctx, mx.data(), maxrun, sizeof(unsigned int) * nkeys);
  // streams: one per (CTA, warp), group-aligned; segments chunk-aligned
  std::vector<long long> useg(nkeys), seg_base(nkeys), nch(nkeys), off((size_t)P * kNW * (Bh + 1));
  long long u_acc = 0, p_acc = 0;
  for (int64_t sw = 0; sw < (int64_t)P * kNW; ++sw) {
    for (int b = 0; b < Bh; ++b) {
      const int64_t k = sw * Bh + b;
      useg[k] = u_acc;
      u_acc += (long long)h[k];
      // every block of the CTA's column part holds at least one chunk (all
      // padding if need be): its first chunk carries the block-boundary flag
      const int part = (int)((sw / kNW) % S);
      const bool exists = b < (part == 0 ? nb0 : nb1);
      nch[k] = exists ? std::max<long long>({1LL, ((long long)h[k] + 31) / 32, (long long)mx[k]}) : 0;
      seg_base[k] = p_acc;
      off[(size_t)sw * (Bh + 1) + b] = p_acc;
      p_acc += 32 * nch[k];
    }
    off[(size_t)sw * (Bh + 1) + Bh] = p_acc;
    p_acc = (p_acc + kGE - 1) / kGE * kGE;  // next stream starts on a group
  }
  const int64_t total = p_acc + kGE;  // an empty last stream still loads (and ignores) one group
  if (std::getenv("SPK_DEBUG_BLOCKED"))
    std::fprintf(stderr, "[blocked] n_out %lld S %d B %d W %d entries %lld padded %lld (x%.3f) max_rows %d\n",
                 (long long)n_out, S, B, W, (long long)m, (long long)p_acc, (double)p_acc / std::max<int64_t>(m, 1),
                 max_rows);
  DBuf d_useg, d_seg, d_nch;
  upload(ctx, d_useg, useg.data(), sizeof(long long) * nkeys);
  upload(ctx, d_seg, seg_base.data(), sizeof(long long) * nkeys);
  upload(ctx, d_nch, nch.data(), sizeof(long long) * nkeys);
  upload(ctx, out.off, off.data(), sizeof(long long) * off.size());
  out.packed.alloc(sizeof(uint32_t) * total);
  out.val.alloc((size_t)vbytes * total);
  const uint32_t pad = (uint32_t)max_rows << 16;  // padding entry: the half's sink row, column 0, value 0
  fill_u32<<<grid_cap(ctx, total), 256, 0, s>>>(out.packed.as<uint32_t>(), total, pad);
  first_chunk_kernel<<<grid_cap(ctx, nkeys * 32), 256, 0, s>>>(nkeys, d_seg.as<long long>(), d_nch.as<long long>(), pad,
                                                                out.packed.as<uint32_t>());
  ctx->launches += 2;
  SPK_CUDA(cudaMemsetAsync(out.val.p, 0, out.val.bytes, s));
  if (m > 0) {
    DBuf& newpos = tmp_buf(ctx, 9, sizeof(int) * mm);
    SPK_CUDA(cudaMemsetAsync(newpos.p, 0xff, sizeof(int) * mm, s));
    phase("runs + host offsets");
    const bool direct = ctx->blocked_spread == 1;
    if (ctx->blocked_spread) {
      DBuf& colc = tmp_buf(ctx, 10, mm);
      colclass_kernel<<<grid_cap(ctx, m), 256, 0, s>>>(perm.as<uint32_t>(), idx_d.as<uint32_t>(), W, (uint32_t)split, m,
                                                       colc.as<unsigned char>());
      if (direct) {
        DBuf stats;
        const bool want = std::getenv("SPK_DEBUG_BLOCKED") != nullptr;
        if (want) {
          stats.alloc(sizeof(unsigned long long) * 8);
          SPK_CUDA(cudaMemsetAsync(stats.p, 0, stats.bytes, s));
        }
        color_warp_kernel<512, 32, 8, false><<<(int)((nkeys + 7) / 8), 32 * 8, 0, s>>>(
            nkeys, d_useg.as<long long>(), hist.as<unsigned long long>(), d_nch.as<long long>(), rl.as<uint32_t>(),
            colc.as<unsigned char>(), d_seg.as<long long>(), pad >> 16, newpos.as<int>(), out.packed.as<uint32_t>(),
            want ? stats.as<unsigned long long>() : nullptr);
        color_warp_kernel<1024, 64, 4, true><<<(int)((nkeys + 3) / 4), 32 * 4, 0, s>>>(
            nkeys, d_useg.as<long long>(), hist.as<unsigned long long>(), d_nch.as<long long>(), rl.as<uint32_t>(),
            colc.as<unsigned char>(), d_seg.as<long long>(), pad >> 16, newpos.as<int>(), out.packed.as<uint32_t>(),
            want ? stats.as<unsigned long long>() : nullptr);
        ++ctx->launches;
        if (want) {
          unsigned long long hs[8];
          download(ctx, hs, stats, sizeof hs);
          std::fprintf(stderr, "[blocked] colouring: %llu segments placed, %llu fell back (path %llu, no room %llu); "
                       "%llu entries beyond their class's colours, %llu evicted after a flip\n",
                       hs[0], hs[1], hs[2], hs[3], hs[4], hs[5]);
        }
      } else
        slot_warp_kernel<<<(int)((nkeys + kSlotWarps - 1) / kSlotWarps), 32 * kSlotWarps, 0, s>>>(
            nkeys, d_useg.as<long long>(), hist.as<unsigned long long>(), d_nch.as<long long>(), rl.as<uint32_t>(),
            colc.as<unsigned char>(), start.as<uint32_t>(), runlen.as<uint32_t>(), newpos.as<int>());
      ++ctx->launches;
    }
    if (vbytes == 4)
      place_kernel<float><<<grid_cap(ctx, m), 256, 0, s>>>(
          keys_s.as<uint32_t>(), perm.as<uint32_t>(), rl.as<uint32_t>(), start.as<uint32_t>(), runlen.as<uint32_t>(),
          d_useg.as<long long>(), d_seg.as<long long>(), d_nch.as<long long>(), idx_d.as<uint32_t>(),
          val_d.as<float>(), W, (uint32_t)split, m, newpos.as<int>(), direct, out.packed.as<uint32_t>(), out.val.as<float>());
    else
      place_kernel<double><<<grid_cap(ctx, m), 256, 0, s>>>(
          keys_s.as<uint32_t>(), perm.as<uint32_t>(), rl.as<uint32_t>(), start.as<uint32_t>(), runlen.as<uint32_t>(),
          d_useg.as<long long>(), d_seg.as<long long>(), d_nch.as<long long>(), idx_d.as<uint32_t>(),
          val_d.as<double>(), W, (uint32_t)split, m, newpos.as<int>(), direct, out.packed.as<uint32_t>(), out.val.as<double>());
    ctx->launches += ctx->blocked_spread ? 2 : 1;
  }
  SPK_CUDA(cudaGetLastError());
  SPK_CUDA(cudaStreamSynchronize(s));
  phase("spread + place");
  if (const char* dump = std::getenv("SPK_DUMP_BLOCKED")) {  // layout diagnostics: the head of the key stream
    std::vector<uint32_t> hk((size_t)std::min<int64_t>(total, 1 << 21));
    download(ctx, hk.data(), out.packed, hk.size() * 4);
    if (FILE* f = std::fopen(dump, "wb")) {
      std::fwrite(hk.data(), 4, hk.size(), f);
      std::fclose(f);
    }
  }
  out.max_rows = max_rows;
  out.padded = p_acc;
  out.cta_entries.assign(P, 0);
  for (int c = 0; c < P; ++c)
    for (int wv = 0; wv < kNW; ++wv) {
      const size_t o = ((size_t)c * kNW + wv) * (Bh + 1);
      out.cta_entries[c] += off[o + Bh] - off[o];
    }
  out.h.P = P;
  out.h.S = S;
  out.h.B = B;
  out.h.split = split;
  out.h.Bh = Bh;
  out.h.W = W;
  out.h.n_out = n_out;
  out.h.n_in = n_in;
  out.h.slab_row0 = out.slab_row0.as<int>();
  out.h.off = out.off.as<long long>();
  out.h.packed = out.packed.as<uint32_t>();
  out.h.val = out.val.p;
  return true;
}

namespace {

// dynamic shared memory per CTA: 227 KB minus the loop kernel's static use
constexpr size_t kSmemBudget = 232448 - 1024;

template <class VT, int S, int STG, bool CL = false>
void launch_blocked(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy,
                    LoopState& st, LoopOut& out) {
  const int64_t n = sk->n;
  BlockedOp<VT, S, STG, CL> op{};
  op.L[0] = sk->blk_rows->h;
  op.L[1] = sk->blk_cols->h;
  op.n = n;
  op.acc_rows = std::max(sk->blk_rows->max_rows, sk->blk_cols->max_rows);
  LoopWs& W = sk->ws;
  W.scalar.ensure(sizeof(unsigned int) * 2);
  SPK_CUDA(cudaMemsetAsync(W.scalar.p, 0, sizeof(unsigned int) * 2, ctx->stream));
  op.fault = W.scalar.as<unsigned int>();
  static const bool trace = std::getenv("SPK_TRACE_BLOCKED") != nullptr;
  DBuf tbuf;
  if (trace) {
    tbuf.alloc(sizeof(unsigned long long) * 4 * 2 * op.L[0].P * 24);
    SPK_CUDA(cudaMemsetAsync(tbuf.p, 0, tbuf.bytes, ctx->stream));
    op.trace = tbuf.as<unsigned long long>();
  }
  const int Q = op.L[0].P / S;
  if (S == 2 && !CL) {
    W.xchg.ensure(sizeof(double) * n);
    W.pair.ensure(sizeof(unsigned int) * Q);
    SPK_CUDA(cudaMemsetAsync(W.pair.p, 0, sizeof(unsigned int) * Q, ctx->stream));
    op.xchg = W.xchg.as<double>();
    op.pair = W.pair.as<unsigned int>();
  }
  W.row_ne.ensure(n);
  W.col_ne.ensure(n);
  SPK_CUDA(cudaMemcpyAsync(W.row_ne.p, sk->cov_row.p, n, cudaMemcpyDeviceToDevice, ctx->stream));
  SPK_CUDA(cudaMemcpyAsync(W.col_ne.p, sk->cov_col.p, n, cudaMemcpyDeviceToDevice, ctx->stream));
  loopcore::run_core<false>(ctx, op, n, W, sk->cov_empty_rows, sk->cov_empty_cols, cfg, exponent, policy, st,
                            /*useful_blocks=*/op.L[0].P, out, /*exact_grid=*/op.L[0].P, op.smem_bytes());
  if (trace) {  // per (iteration, half, CTA): half start, 15 warps' stream ends, finalize end (ns)
    std::vector<unsigned long long> h(tbuf.bytes / 8);
    download(ctx, h.data(), tbuf, tbuf.bytes);
    const int P = op.L[0].P;
    for (int it = 0; it < 4; ++it)
      for (int role = 0; role < 2; ++role) {
        unsigned long long t0 = ~0ull, t1 = 0, smin = ~0ull, smax = 0, fmax = 0;
        long double smean = 0;
        int cntw = 0;
        for (int c = 0; c < P; ++c) {
          const unsigned long long* e = h.data() + (((size_t)it * 2 + role) * P + c) * 24;
          if (!e[0]) continue;
          t0 = std::min(t0, e[0]);
          t1 = std::max(t1, e[0]);
          fmax = std::max(fmax, e[19]);
          for (int w = 0; w < kNW; ++w)
            if (e[1 + w]) {
              smin = std::min(smin, e[1 + w]);
              smax = std::max(smax, e[1 + w]);
              smean += (long double)(e[1 + w] - e[0]);
              ++cntw;
            }
        }
        if (t0 == ~0ull) continue;
        std::fprintf(stderr,
                     "[trace] it %d half %d: start spread %.1f us, stream end min %.1f mean %.1f max %.1f us, "
                     "finalize end %.1f us\n",
                     it + 1, role, (t1 - t0) * 1e-3, (smin - t0) * 1e-3, (double)(smean / cntw) * 1e-3,
                     (smax - t0) * 1e-3, (fmax - t0) * 1e-3);
        // per-CTA phase durations averaged: stream end (last warp) -> released, -> xchg written, -> pair met, -> final
        double d1 = 0, d2 = 0, d3 = 0, d4 = 0;
        int nc = 0;
        for (int c = 0; c < P; ++c) {
          const unsigned long long* e = h.data() + (((size_t)it * 2 + role) * P + c) * 24;
          if (!e[0] || !e[16]) continue;
          unsigned long long se = 0;
          for (int w = 0; w < kNW; ++w) se = std::max(se, e[1 + w]);
          d1 += (double)(e[16] - se);
          if (e[17]) d2 += (double)(e[17] - e[16]);
          d3 += (double)(e[18] - (e[17] ? e[17] : e[16]));
          d4 += (double)(e[19] - e[18]);
          ++nc;
        }
        {  // stream time per CTA against its padded entries (and its slowest warp against the mean warp)
          const std::vector<long long>& ce = role == 0 ? sk->blk_rows->cta_entries : sk->blk_cols->cta_entries;
          double sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0, wspread = 0;
          int cnt = 0;
          for (int c = 0; c < P && c < (int)ce.size(); ++c) {
            const unsigned long long* e = h.data() + (((size_t)it * 2 + role) * P + c) * 24;
            if (!e[0]) continue;
            unsigned long long se = 0, smn = ~0ull;
            for (int w = 0; w < kNW; ++w)
              if (e[1 + w]) {
                se = std::max(se, e[1 + w]);
                smn = std::min(smn, e[1 + w]);
              }
            const double x = (double)ce[c], y = (double)(se - e[0]);
            sx += x; sy += y; sxx += x * x; syy += y * y; sxy += x * y;
            wspread += (double)(se - smn);
            ++cnt;
          }
          const double cov = sxy / cnt - sx / cnt * sy / cnt, vx = sxx / cnt - sx / cnt * sx / cnt,
                       vy = syy / cnt - sy / cnt * sy / cnt;
          std::fprintf(stderr, "[trace]   CTA stream time vs padded entries: corr %.3f, entries cv %.4f, time cv %.4f; "
                       "warp spread in a CTA %.1f us\n", cov / std::sqrt(vx * vy + 1e-30), std::sqrt(vx) / (sx / cnt),
                       std::sqrt(vy) / (sy / cnt), wspread / cnt * 1e-3);
        }
        if (it == 3) {  // are the slow CTAs the same from iteration to iteration? (SM position vs data)
          std::vector<std::pair<double, int>> tm;
          double sa = 0, sb = 0, saa = 0, sbb = 0, sab = 0;
          for (int c = 0; c < P; ++c) {
            const unsigned long long* e3 = h.data() + (((size_t)3 * 2 + role) * P + c) * 24;
            const unsigned long long* e2 = h.data() + (((size_t)2 * 2 + role) * P + c) * 24;
            unsigned long long s3 = 0, s2 = 0;
            for (int w = 0; w < kNW; ++w) {
              s3 = std::max(s3, e3[1 + w]);
              s2 = std::max(s2, e2[1 + w]);
            }
            const double a = (double)(s3 - e3[0]), b = (double)(s2 - e2[0]);
            tm.push_back({a, c});
            sa += a; sb += b; saa += a * a; sbb += b * b; sab += a * b;
          }
          const double ca = sab / P - sa / P * sb / P, va = saa / P - sa / P * sa / P, vb = sbb / P - sb / P * sb / P;
          std::sort(tm.begin(), tm.end());
          std::fprintf(stderr, "[trace]   per-CTA stream time, iteration 4 vs 3: corr %.3f; slowest CTAs (cta:smid:us):",
                       ca / std::sqrt(va * vb + 1e-30));
          for (int k = 0; k < 12; ++k) {
            const int c = tm[P - 1 - k].second;
            std::fprintf(stderr, " %d:%llu:%.1f", c, h[(((size_t)3 * 2 + role) * P + c) * 24 + 20], tm[P - 1 - k].first * 1e-3);
          }
          std::fprintf(stderr, "; fastest:");
          for (int k = 0; k < 12; ++k) {
            const int c = tm[k].second;
            std::fprintf(stderr, " %d:%llu:%.1f", c, h[(((size_t)3 * 2 + role) * P + c) * 24 + 20], tm[k].first * 1e-3);
          }
          std::fprintf(stderr, "\n");
        }
        std::fprintf(stderr, "[trace]   per CTA: release %.2f us, xchg %.2f us, pair wait %.2f us, finalize %.2f us\n",
                     d1 / nc * 1e-3, d2 / nc * 1e-3, d3 / nc * 1e-3, d4 / nc * 1e-3);
      }
  }
  unsigned int fw[2] = {0u, 0u};
  download(ctx, fw, W.scalar, sizeof fw);
  if (fw[0]) {
    // code: 1 producer / 2-4 consumer barrier wait / 5 pair exchange timed out; then half and block
    const std::string msg = "blocked loop: a tile barrier timed out (site " + std::to_string(fw[0] >> 28) +
                            ", half " + std::to_string((fw[0] >> 24) & 15) + ", block " +
                            std::to_string(fw[0] & 0xffffff) + ", CTA " + std::to_string(fw[1]) + ")";
    fail_device(msg.c_str(), cudaErrorLaunchTimeout);
  }
}

// Ring depths: S = 1 keeps 4 tiles in flight; S = 2 doubles the accumulator
// rows per CTA and keeps 3.
constexpr int kStg1 = 4, kStg2 = 3;

// The cluster variant needs every CTA pair co-resident as a 2-CTA cluster
// (a GPC with an odd number of free SMs loses one); else the L2 swap is used.
template <class VT>
bool cluster_pairs_fit(spk_ctx* ctx, spk_sketch* sk) {
  if (!ctx->blocked_cluster) return false;
  const int P = sk->blk_rows->h.P;
  BlockedOp<VT, 2, kStg2, true> probe{};
  probe.acc_rows = std::max(sk->blk_rows->max_rows, sk->blk_cols->max_rows);
  const size_t smem = probe.smem_bytes();
  auto kern = loopcore::loop_kernel<false, false, BlockedOp<VT, 2, kStg2, true>>;
  loopcore::allow_max_dyn_smem((const void*)kern);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(P);
  lc.blockDim = dim3(kThreadsBlocked);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)kern, &lc) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return nclusters >= P / 2;
}

template <class VT>
bool run_blocked_t(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy,
                   LoopState& st, LoopOut& out) {
  const int64_t n = sk->n;
  if (!sk->blocked_tried) {
    sk->blocked_tried = true;
    const int vb = sizeof(VT);
    const int W = std::min(kTileW, std::max(16, ctx->blocked_max_w));
    // S = 2 when the pair split fits (even SM count, slab accumulators in
    // shared memory); else one CTA per slab
    static const bool dbg = std::getenv("SPK_DEBUG_TIMING") != nullptr;
    Timer tb(ctx->stream);
    for (int S = (ctx->blocked_split == 1 ? 1 : 2); S >= 1; --S) {
      if (S == 2 && ctx->num_sms < 2) continue;
      const int P = (ctx->num_sms / S) * S;
      auto R = std::make_unique<BlockedHost>(), C = std::make_unique<BlockedHost>();
      if (!build_blocked(ctx, P, S, W, n, n, sk->nnz, sk->row_ptr, sk->col_idx, sk->values, vb, *R) ||
          !build_blocked(ctx, P, S, W, n, n, sk->nnz, sk->col_ptr, sk->row_idx, sk->values_t, vb, *C))
        continue;
      const int acc_rows = std::max(R->max_rows, C->max_rows);
      const size_t smem = S == 2 ? BlockedOp<VT, 2, kStg2>{{}, 0, acc_rows}.smem_bytes()
                                 : BlockedOp<VT, 1, kStg1>{{}, 0, acc_rows}.smem_bytes();
      // auto mode keeps the CSR loop when rows are too few per warp to fill
      // conflict-free chunks (padding would outweigh the staged gathers)
      // (config 5, n = 5e4: 41% padding and still 27.0k against the CSR loop's 16.5k iterations/s;
      // the stream time grows with the padded entries, so ~2.3x would break even)
      const bool dense_pad = ctx->use_blocked == 2 && (double)(R->padded + C->padded) > 1.8 * 2.0 * (double)sk->nnz;
      if (smem <= kSmemBudget && !dense_pad) {
        sk->blk_rows = std::move(R);
        sk->blk_cols = std::move(C);
        break;
      }
      if (ctx->blocked_split == 2) break;
    }
    if (dbg) std::fprintf(stderr, "[timing] blocked layouts %.4f s\n", tb.stop());
  }
  if (!sk->blk_rows) return false;
  if (sk->blk_rows->h.S == 2 && cluster_pairs_fit<VT>(ctx, sk))
    launch_blocked<VT, 2, kStg2, true>(ctx, sk, cfg, exponent, policy, st, out);
  else if (sk->blk_rows->h.S == 2)
    launch_blocked<VT, 2, kStg2>(ctx, sk, cfg, exponent, policy, st, out);
  else launch_blocked<VT, 1, kStg1>(ctx, sk, cfg, exponent, policy, st, out);
  return true;
}

}  // namespace

// ---- sharded half-steps (shard.cu's state machine, this file's operator) -----------

namespace {

template <class VT, int S, int STG, bool CL>
__global__ void __launch_bounds__(kThreadsBlocked, 1) shard_half_kernel(shard::HalfArgs A, BlockedOp<VT, S, STG, CL> op) {
  __shared__ shard::State St;
  if (threadIdx.x == 0) {
    St = *A.st_in;
    shard::decide<false>(A, St);
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) *A.st_out = St;
  if (St.stopped) return;  // the same decision in every CTA (same gathered tails)
  double err = 0.0;
  long long masks = 0;
  if (A.half == 0)
    op.template half<0, false, false>(A.x, A.w, A.old, A.out, A.ne, A.dyn, A.exponent, A.policy, (int)A.t, A.flag,
                                      nullptr, err, masks);
  else
    op.template half<1, false, false>(A.x, A.w, A.old, A.out, A.ne, A.dyn, A.exponent, A.policy, (int)A.t, A.flag,
                                      nullptr, err, masks);
  shard::finish_half(A, err, masks);
}

template <class VT>
void launch_shard_half(spk_ctx* ctx, const shard::HalfArgs& A, shard::BlockedShard& B) {
  const BlockedHalf& h = B.R->h;
  const int acc_rows = std::max(B.R->max_rows, B.C->max_rows);
  if (h.S == 2) {  // CTA pairs as 2-CTA clusters (independent clusters: no co-residency needed)
    BlockedOp<VT, 2, kStg2, true> op{};
    op.L[0] = B.R->h;
    op.L[1] = B.C->h;
    op.n = h.n_out;
    op.acc_rows = acc_rows;
    op.fault = B.fault.as<unsigned int>();
    op.fresh = true;
    auto kern = shard_half_kernel<VT, 2, kStg2, true>;
    const size_t smem = op.smem_bytes();
    loopcore::allow_max_dyn_smem((const void*)kern);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(h.P);
    lc.blockDim = dim3(kThreadsBlocked);
    lc.dynamicSmemBytes = smem;
    lc.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    shard::HalfArgs a = A;
    void* args[] = {&a, &op};
    SPK_CUDA(cudaLaunchKernelExC(&lc, (const void*)kern, args));
  } else {
    BlockedOp<VT, 1, kStg1> op{};
    op.L[0] = B.R->h;
    op.L[1] = B.C->h;
    op.n = h.n_out;
    op.acc_rows = acc_rows;
    op.fault = B.fault.as<unsigned int>();
    op.fresh = true;
    auto kern = shard_half_kernel<VT, 1, kStg1, false>;
    const size_t smem = op.smem_bytes();
    loopcore::allow_max_dyn_smem((const void*)kern);
    kern<<<h.P, kThreadsBlocked, smem, ctx->stream>>>(A, op);
  }
  ++ctx->launches;
  SPK_CUDA(cudaGetLastError());
}

}  // namespace

namespace shard {

bool blocked_shard_build(spk_ctx* ctx, int64_t m_own, int64_t n_in, int64_t nnz_r, const DBuf& row_ptr,
                         const DBuf& col_idx, const DBuf& vals, int64_t nnz_c, const DBuf& col_ptr,
                         const DBuf& row_idx, const DBuf& vals_t, int vbytes, BlockedShard& out) {
  const int W = std::min(kTileW, std::max(16, ctx->blocked_max_w));
  for (int S = (ctx->blocked_split == 1 || !ctx->blocked_cluster ? 1 : 2); S >= 1; --S) {
    if (S == 2 && ctx->num_sms < 2) continue;
    const int P = (ctx->num_sms / S) * S;
    auto R = std::make_unique<BlockedHost>(), C = std::make_unique<BlockedHost>();
    if (!build_blocked(ctx, P, S, W, m_own, n_in, nnz_r, row_ptr, col_idx, vals, vbytes, *R) ||
        !build_blocked(ctx, P, S, W, m_own, n_in, nnz_c, col_ptr, row_idx, vals_t, vbytes, *C))
      continue;
    const int acc_rows = std::max(R->max_rows, C->max_rows);
    const size_t smem = S == 2 ? (vbytes == 4 ? BlockedOp<float, 2, kStg2, true>{{}, 0, acc_rows}.smem_bytes()
                                              : BlockedOp<double, 2, kStg2, true>{{}, 0, acc_rows}.smem_bytes())
                               : (vbytes == 4 ? BlockedOp<float, 1, kStg1>{{}, 0, acc_rows}.smem_bytes()
                                              : BlockedOp<double, 1, kStg1>{{}, 0, acc_rows}.smem_bytes());
    if (smem > kSmemBudget) continue;
    out.R = std::move(R);
    out.C = std::move(C);
    out.vbytes = vbytes;
    out.fault.alloc(sizeof(unsigned int) * 2);
    SPK_CUDA(cudaMemsetAsync(out.fault.p, 0, out.fault.bytes, ctx->stream));
    return true;
  }
  return false;
}

void blocked_shard_half(spk_ctx* ctx, const HalfArgs& A, BlockedShard& B) {
  if (B.vbytes == 4) launch_shard_half<float>(ctx, A, B);
  else launch_shard_half<double>(ctx, A, B);
}

}  // namespace shard

bool run_blocked(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy, LoopState& st,
                 LoopOut& out) {
  if (sk->value_type == SPK_VALUES_F32) return run_blocked_t<float>(ctx, sk, cfg, exponent, policy, st, out);
  return run_blocked_t<double>(ctx, sk, cfg, exponent, policy, st, out);
}

}  // namespace spk
