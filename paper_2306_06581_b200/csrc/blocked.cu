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
//   output atoms (this half's rows) are cut into P = #SMs slabs of ~equal
//   entry count, one per persistent CTA, each slab into 16 warp ranges;
//   input atoms are cut into B blocks of W = 8192 atoms (one 64 KB x tile).
//   Entries are ordered (slab, warp, block, row, col): each warp's whole half
//   is ONE contiguous stream, and inside a row the columns still ascend, so
//   every row is summed in the reference's j order (spmv,
//   proj/src/sparsify.cpp:203-213; spmv_t :215-226 on the CSC). Each
//   (slab, warp, block) segment is padded to 32 entries. An entry is packed
//   (row_local << 16 | col_local) + value: no more bytes than a CSR entry.
// Half-step (inside the persistent loop, loop_core.cuh), 17 warps per CTA:
//   * producer warp: cp.async.bulk (TMA) of x tile b into stage b%2 as soon as
//     every consumer released stage b-2 (empty mbarrier) -- 64 KB copies, the
//     size at which 1-D bulk copies stream at full rate on B200
//     (profiles/microbench/r1_tma_stream_b200.txt: 8 KB 2.3 TB/s, 64 KB 7.1 TB/s);
//   * 16 consumer warps stream their entries with coalesced loads, 256
//     entries double-buffered in registers ahead of use (independent of the
//     tile pipeline), gather x from the shared tile, and fold each 32-entry
//     chunk with a head-mask segmented scan (usually one shuffle step) into
//     their own rows' shared accumulators (no atomics, deterministic).
// L2->SM traffic per half: the entry stream + P tiles of x, instead of one
// random 32-byte sector per entry.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "internal.h"
#include "loop_core.cuh"

namespace spk {

namespace {

constexpr int kNW = 16;                 // consumer warps per CTA
constexpr int kThreadsBlocked = 32 * (kNW + 1);
constexpr int kTileW = 8192;            // x tile: 64 KB of fp64
constexpr int kGroup = 8;               // chunks of 32 entries per prefetch group
constexpr uint32_t kPad = 0xffffffffu;  // padding entry (never a valid packed value)

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
// Bounded wait: false after ~2^24 polls (a lost transaction must not hang the
// GPU; the caller records a fault and the host raises it).
__device__ __forceinline__ bool mbar_wait(uint64_t* bar, uint32_t parity) {
  for (int spin = 0; spin < (1 << 24); ++spin) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return true;
  }
  return false;
}
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <class VT>
struct BlockedOp {
  static constexpr int kThreads = kThreadsBlocked;
  static constexpr int kMinBlocks = 1;  // one CTA per SM: full register file, ~200 KB shared
  BlockedHalf L[2];
  int64_t n;
  int acc_rows;  // shared accumulator capacity (max rows of a slab over both halves)
  unsigned int* fault;

  __host__ __device__ size_t head_bytes() const { return align16((size_t)acc_rows * 8) + 64; }
  size_t smem_bytes() const { return head_bytes() + (size_t)2 * kTileW * 8; }

  // One 32-entry chunk: gather, segmented scan by row, tail add.
  __device__ __forceinline__ void fold(uint32_t u, double v, const double* xs, double* acc, int lane,
                                       unsigned upto) const {
    if (u != kPad) v *= xs[u & 0xffffu];
    else v = 0.0;
    const uint32_t rl = u >> 16;
    const uint32_t up = __shfl_up_sync(0xffffffffu, rl, 1);
    const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || up != rl);
    const int sstart = 31 - __clz(heads & upto);
    for (int d = 1; d < 32; d <<= 1) {
      if (!__any_sync(0xffffffffu, lane - d >= sstart)) break;
      const double vo = __shfl_up_sync(0xffffffffu, v, d);
      if (lane - d >= sstart) v += vo;
    }
    const bool tail = lane == 31 || ((heads >> (lane + 1)) & 1u);
    if (tail && u != kPad) acc[rl] += v;
  }

  template <int ROLE, bool LOG, bool DET>
  __device__ void half(const double* x, const double* wgt, const double* old, double* out, unsigned char* ne,
                       int* dyn, double exponent, int policy, int t, unsigned long long* flag, double* absdiff,
                       double& err, long long& masks) const {
    extern __shared__ __align__(128) unsigned char dsm[];
    double* acc = reinterpret_cast<double*>(dsm);
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm + align16((size_t)acc_rows * 8));
    uint64_t* empty = full + 2;
    double* tiles = reinterpret_cast<double*>(dsm + head_bytes());

    const BlockedHalf& H = L[ROLE];
    const int p = blockIdx.x;
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const VT* gval = static_cast<const VT*>(H.val);
    const int r0 = H.slab_row0[p];
    const int nrows = H.slab_row0[p + 1] - r0;
    const int B = H.B;

    if (threadIdx.x == 0) {
      mbar_init(&full[0], 1);
      mbar_init(&full[1], 1);
      mbar_init(&empty[0], kNW);
      mbar_init(&empty[1], kNW);
      fence_mbar_init();
    }
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) acc[r] = 0.0;
    __syncthreads();

    if (w == kNW) {
      // ---- producer warp: x tiles, two stages ----
      if (lane == 0) {
        fence_proxy_async();  // x was written with generic stores before the grid barrier
        for (int b = 0; b < B; ++b) {
          const int s = b & 1;
          if (b >= 2 && !mbar_wait(&empty[s], (uint32_t)(((b - 2) >> 1) & 1))) atomicExch(fault, 1u);
          const int64_t c0 = (int64_t)b * H.W;
          const int64_t cnt = min((int64_t)H.W, H.n_in - c0);
          const uint32_t bytes = (uint32_t)align16((size_t)cnt * 8);
          mbar_arrive_expect_tx(&full[s], bytes);
          bulk_copy_g2s(tiles + (size_t)s * kTileW, x + c0, bytes, &full[s]);
        }
      }
    } else {
      // ---- consumer warps: one contiguous entry stream per warp ----
      const long long* ofs = H.off + ((int64_t)p * kNW + w) * (B + 1);  // block starts, padded, [B] = end
      const long long sbeg = ofs[0], send = ofs[B];
      const unsigned upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
      int cb = 0;  // current block
      long long cb_end = ofs[1];
      if (!mbar_wait(&full[0], 0u)) atomicExch(fault, 1u);
      uint32_t ua[kGroup], ub[kGroup];
      VT va[kGroup], vb[kGroup];
      // two register groups of 8 chunks: load group g+1 while folding group g
#define SPK_LOAD(G0, UU, VV)                                     \
  _Pragma("unroll") for (int k = 0; k < kGroup; ++k) {           \
    const long long e = (G0) + 32 * k + lane;                    \
    UU[k] = e < send ? __ldcs(H.packed + e) : kPad;              \
    VV[k] = e < send ? __ldcs(gval + e) : (VT)0;                 \
  }
#define SPK_CONSUME(G0, UU, VV)                                                          \
  _Pragma("unroll") for (int k = 0; k < kGroup; ++k) {                                   \
    const long long c = (G0) + 32 * k;                                                   \
    if (c < send) { /* warp-uniform; no break so the group stays in registers */        \
      while (c >= cb_end) { /* leave block cb (release its tile), enter the next */      \
        __syncwarp();                                                                    \
        if (lane == 0) mbar_arrive(&empty[cb & 1]);                                      \
        ++cb;                                                                            \
        cb_end = ofs[cb + 1];                                                            \
        if (!mbar_wait(&full[cb & 1], (uint32_t)((cb >> 1) & 1))) atomicExch(fault, 1u); \
      }                                                                                  \
      fold(UU[k], (double)VV[k], tiles + (size_t)(cb & 1) * kTileW, acc, lane, upto);    \
    }                                                                                    \
  }
      const long long step = 32LL * kGroup;
      long long g = sbeg;
      if (g < send) { SPK_LOAD(g, ua, va) }
      while (g < send) {
        const long long g1 = g + step;
        if (g1 < send) { SPK_LOAD(g1, ub, vb) }
        SPK_CONSUME(g, ua, va)
        g = g1;
        if (g >= send) break;
        const long long g2 = g + step;
        if (g2 < send) { SPK_LOAD(g2, ua, va) }
        SPK_CONSUME(g, ub, vb)
        g = g2;
      }
#undef SPK_LOAD
#undef SPK_CONSUME
      // release the remaining blocks in order (tile present before release)
      for (;;) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cb & 1]);
        if (++cb >= B) break;
        if (!mbar_wait(&full[cb & 1], (uint32_t)((cb >> 1) & 1))) atomicExch(fault, 1u);
      }
    }
    __syncthreads();
    // ---- finalize this slab's atoms ----
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
      const int64_t i = r0 + r;
      const double o = __ldcg(old + i);
      if (!ne[i]) {
        out[i] = o;
        continue;
      }
      err += loopcore::finalize_atom<LOG>(i, acc[r], o, wgt[i], exponent, policy, t, ne, dyn, out, flag, masks);
    }
    __syncthreads();
  }
};

// ---- layout builder --------------------------------------------------------------

// key = ((slab * NW + warp) * B + block): the warp's whole stream is contiguous
__global__ void key_kernel(const long long* ptr, const uint32_t* idx, int64_t n_out, const int* slab_of,
                           const unsigned char* warp_of, int W, int B, uint32_t* keys) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_out; i += nw) {
    const uint32_t base = ((uint32_t)slab_of[i] * kNW + warp_of[i]) * (uint32_t)B;
    for (long long q = ptr[i] + lane; q < ptr[i + 1]; q += 32) keys[q] = base + idx[q] / (uint32_t)W;
  }
}

// Sorted position q (key k) -> padded destination seg_base[k] + (q - useg[k]).
template <class VT>
__global__ void pack_kernel(const uint32_t* keys_s, const uint32_t* perm, const uint32_t* idx, const VT* val,
                            const uint32_t* rows_of_pos, const int* slab_row0_of_row, const long long* useg,
                            const long long* seg_base, int W, int64_t m, uint32_t* packed, VT* vout) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys_s[q];
    const long long dst = seg_base[k] + (q - useg[k]);
    const uint32_t src = perm[q];
    const uint32_t i = rows_of_pos[src];
    const uint32_t rl = i - (uint32_t)slab_row0_of_row[i];
    const uint32_t cl = idx[src] % (uint32_t)W;
    packed[dst] = (rl << 16) | cl;
    vout[dst] = val[src];
  }
}

__global__ void rows_of_pos_kernel(const long long* ptr, int64_t n, uint32_t* rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw)
    for (long long p = ptr[i] + lane; p < ptr[i + 1]; p += 32) rows[p] = (uint32_t)i;
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

// Build one half's layout from (ptr, idx, val). Returns false when the shape
// does not fit (rows per slab >= 2^16).
bool build_blocked(spk_ctx* ctx, int P, int W, int64_t n_out, int64_t n_in, int64_t m, const DBuf& ptr_d,
                   const DBuf& idx_d, const DBuf& val_d, int vbytes, BlockedHost& out) {
  std::vector<long long> ptr(n_out + 1);
  download(ctx, ptr.data(), ptr_d, sizeof(long long) * (n_out + 1));
  std::vector<int> slab_row0(P + 1);
  slab_row0[0] = 0;
  for (int k = 1; k < P; ++k) {
    const long long target = (long long)((double)m * k / P);
    int r = (int)(std::lower_bound(ptr.begin(), ptr.end(), target) - ptr.begin());
    slab_row0[k] = std::max<int>(std::min<int64_t>(r, n_out), slab_row0[k - 1]);
  }
  slab_row0[P] = (int)n_out;
  int max_rows = 0;
  for (int k = 0; k < P; ++k) max_rows = std::max(max_rows, slab_row0[k + 1] - slab_row0[k]);
  if (max_rows >= 65535) return false;
  const int B = (int)((n_in + W - 1) / W);
  std::vector<int> slab_of(n_out), slab_row0_of_row(n_out);
  std::vector<unsigned char> warp_of(n_out);
  for (int k = 0; k < P; ++k) {
    const int a = slab_row0[k], z = slab_row0[k + 1];
    const long long e0 = ptr[a], e1 = ptr[z];
    int prev = a;
    for (int wv = 0; wv < kNW; ++wv) {
      int r_end = z;
      if (wv + 1 < kNW) {
        const long long target = e0 + (long long)((double)(e1 - e0) * (wv + 1) / kNW);
        r_end = std::max(prev, (int)(std::lower_bound(ptr.begin() + a, ptr.begin() + z, target) - ptr.begin()));
      }
      for (int r = prev; r < r_end; ++r) {
        slab_of[r] = k;
        warp_of[r] = (unsigned char)wv;
        slab_row0_of_row[r] = a;
      }
      prev = r_end;
    }
  }
  const int64_t nkeys = (int64_t)P * kNW * B;
  if (nkeys >= (1LL << 32)) return false;
  cudaStream_t s = ctx->stream;
  const int64_t mm = std::max<int64_t>(m, 1);
  DBuf d_slab_of, d_warp_of, d_s0r;
  upload(ctx, d_slab_of, slab_of.data(), sizeof(int) * n_out);
  upload(ctx, d_warp_of, warp_of.data(), n_out);
  upload(ctx, d_s0r, slab_row0_of_row.data(), sizeof(int) * n_out);
  DBuf keys(sizeof(uint32_t) * mm), keys_s(sizeof(uint32_t) * mm), iota(sizeof(uint32_t) * mm),
      perm(sizeof(uint32_t) * mm), rows(sizeof(uint32_t) * mm), hist(sizeof(unsigned long long) * nkeys);
  SPK_CUDA(cudaMemsetAsync(hist.p, 0, hist.bytes, s));
  key_kernel<<<grid_cap(ctx, n_out * 32), 256, 0, s>>>(ptr_d.as<long long>(), idx_d.as<uint32_t>(), n_out,
                                                        d_slab_of.as<int>(), d_warp_of.as<unsigned char>(), W, B,
                                                        keys.as<uint32_t>());
  rows_of_pos_kernel<<<grid_cap(ctx, n_out * 32), 256, 0, s>>>(ptr_d.as<long long>(), n_out, rows.as<uint32_t>());
  iota_u32<<<grid_cap(ctx, m), 256, 0, s>>>(iota.as<uint32_t>(), m);
  key_hist_kernel<<<grid_cap(ctx, m), 256, 0, s>>>(keys.as<uint32_t>(), m, hist.as<unsigned long long>());
  ctx->launches += 4;
  int end_bit = 1;
  while ((int64_t(1) << end_bit) < nkeys) ++end_bit;
  size_t tb = 0;
  SPK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<uint32_t>(), keys_s.as<uint32_t>(),
                                           iota.as<uint32_t>(), perm.as<uint32_t>(), (int)m, 0, end_bit, s));
  ctx->scratch.ensure(tb);
  SPK_CUDA(cub::DeviceRadixSort::SortPairs(ctx->scratch.p, tb, keys.as<uint32_t>(), keys_s.as<uint32_t>(),
                                           iota.as<uint32_t>(), perm.as<uint32_t>(), (int)m, 0, end_bit, s));
  ++ctx->launches;
  // host: each (slab, warp, block) segment padded to 32 entries; per-warp block starts
  std::vector<unsigned long long> h(nkeys);
  download(ctx, h.data(), hist, sizeof(unsigned long long) * nkeys);
  std::vector<long long> useg(nkeys), seg_base(nkeys), off((size_t)P * kNW * (B + 1));
  long long u_acc = 0, p_acc = 0;
  for (int64_t sw = 0; sw < (int64_t)P * kNW; ++sw) {
    for (int b = 0; b < B; ++b) {
      const int64_t k = sw * B + b;
      useg[k] = u_acc;
      seg_base[k] = p_acc;
      off[(size_t)sw * (B + 1) + b] = p_acc;
      u_acc += (long long)h[k];
      p_acc += ((long long)h[k] + 31) & ~31LL;
    }
    off[(size_t)sw * (B + 1) + B] = p_acc;
  }
  const int64_t total = std::max<long long>(p_acc, 32);
  DBuf d_useg, d_seg;
  upload(ctx, d_useg, useg.data(), sizeof(long long) * nkeys);
  upload(ctx, d_seg, seg_base.data(), sizeof(long long) * nkeys);
  upload(ctx, out.off, off.data(), sizeof(long long) * off.size());
  upload(ctx, out.slab_row0, slab_row0.data(), sizeof(int) * (P + 1));
  out.packed.alloc(sizeof(uint32_t) * total);
  out.val.alloc((size_t)vbytes * total);
  SPK_CUDA(cudaMemsetAsync(out.packed.p, 0xff, out.packed.bytes, s));  // padding = kPad
  SPK_CUDA(cudaMemsetAsync(out.val.p, 0, out.val.bytes, s));
  if (vbytes == 4)
    pack_kernel<float><<<grid_cap(ctx, m), 256, 0, s>>>(keys_s.as<uint32_t>(), perm.as<uint32_t>(),
                                                         idx_d.as<uint32_t>(), val_d.as<float>(), rows.as<uint32_t>(),
                                                         d_s0r.as<int>(), d_useg.as<long long>(),
                                                         d_seg.as<long long>(), W, m, out.packed.as<uint32_t>(),
                                                         out.val.as<float>());
  else
    pack_kernel<double><<<grid_cap(ctx, m), 256, 0, s>>>(keys_s.as<uint32_t>(), perm.as<uint32_t>(),
                                                          idx_d.as<uint32_t>(), val_d.as<double>(),
                                                          rows.as<uint32_t>(), d_s0r.as<int>(), d_useg.as<long long>(),
                                                          d_seg.as<long long>(), W, m, out.packed.as<uint32_t>(),
                                                          out.val.as<double>());
  ++ctx->launches;
  SPK_CUDA(cudaGetLastError());
  SPK_CUDA(cudaStreamSynchronize(s));
  out.max_rows = max_rows;
  out.ecap = 0;
  out.h.P = P;
  out.h.B = B;
  out.h.W = W;
  out.h.n_out = n_out;
  out.h.n_in = n_in;
  out.h.slab_row0 = out.slab_row0.as<int>();
  out.h.warp_row0 = nullptr;
  out.h.off = out.off.as<long long>();
  out.h.packed = out.packed.as<uint32_t>();
  out.h.val = out.val.p;
  return true;
}

template <class VT>
bool run_blocked_t(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy,
                   LoopState& st, LoopOut& out) {
  const int64_t n = sk->n;
  const int P = ctx->num_sms;
  const size_t budget = 222 * 1024;  // dynamic shared memory per CTA (static use is ~1 KB)
  if (!sk->blocked_tried) {
    sk->blocked_tried = true;
    const int vb = sizeof(VT);
    const int W = std::min(kTileW, std::max(16, ctx->blocked_max_w));
    auto R = std::make_unique<BlockedHost>(), C = std::make_unique<BlockedHost>();
    if (build_blocked(ctx, P, W, n, n, sk->nnz, sk->row_ptr, sk->col_idx, sk->values, vb, *R) &&
        build_blocked(ctx, P, W, n, n, sk->nnz, sk->col_ptr, sk->row_idx, sk->values_t, vb, *C)) {
      BlockedOp<VT> probe{};
      probe.acc_rows = std::max(R->max_rows, C->max_rows);
      if (probe.smem_bytes() <= budget) {
        sk->blk_rows = std::move(R);
        sk->blk_cols = std::move(C);
      }
    }
  }
  if (!sk->blk_rows) return false;
  BlockedOp<VT> op{};
  op.L[0] = sk->blk_rows->h;
  op.L[1] = sk->blk_cols->h;
  op.n = n;
  op.acc_rows = std::max(sk->blk_rows->max_rows, sk->blk_cols->max_rows);
  LoopWs& W = sk->ws;
  W.scalar.ensure(sizeof(unsigned int));
  SPK_CUDA(cudaMemsetAsync(W.scalar.p, 0, sizeof(unsigned int), ctx->stream));
  op.fault = W.scalar.as<unsigned int>();
  W.row_ne.ensure(n);
  W.col_ne.ensure(n);
  SPK_CUDA(cudaMemcpyAsync(W.row_ne.p, sk->cov_row.p, n, cudaMemcpyDeviceToDevice, ctx->stream));
  SPK_CUDA(cudaMemcpyAsync(W.col_ne.p, sk->cov_col.p, n, cudaMemcpyDeviceToDevice, ctx->stream));
  loopcore::run_core<false>(ctx, op, n, W, sk->cov_empty_rows, sk->cov_empty_cols, cfg, exponent, policy, st,
                            /*useful_blocks=*/P, out, /*exact_grid=*/P, op.smem_bytes());
  unsigned int fault = 0;
  download(ctx, &fault, W.scalar, sizeof fault);
  if (fault) fail_device("blocked loop: a TMA tile never completed", cudaErrorLaunchTimeout);
  return true;
}

bool run_blocked(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy, LoopState& st,
                 LoopOut& out) {
  if (sk->value_type == SPK_VALUES_F32) return run_blocked_t<float>(ctx, sk, cfg, exponent, policy, st, out);
  return run_blocked_t<double>(ctx, sk, cfg, exponent, policy, st, out);
}

}  // namespace spk
