// blocked.cu -- the fast sparse half-step: slab x block sketch layout with the
// scaling vector staged in shared memory by TMA bulk copies (north-star item 3:
// "shared-memory/TMA staging of the gathered scaling vector").
//
// Why: at config 4 (n = 1e6, 1.1e8 entries, columns uniformly random) every
// gathered x[j] of the CSR kernel is a random 8-byte read, i.e. one 32-byte
// L2 sector per entry: 3.5 GB of L2->SM sectors per half, twice the sketch
// stream itself, and the measured bound of the plain kernel.
//
// Layout (built once per sketch, for the CSR and for the CSC mirror):
//   output atoms (rows of this half) are cut into P slabs of ~equal entry
//   count, one per persistent CTA, and each slab into NW warp ranges;
//   input atoms (columns) are cut into B blocks of W (<= 16384) atoms.
//   Entries are ordered (slab, block, warp, row, col) -- inside one row the
//   columns still ascend, so every row is summed in the reference's j order
//   (spmv, proj/src/sparsify.cpp:203-213; spmv_t :215-226 for the CSC).
//   An entry is 8 bytes: packed (row_local << 16 | col_local) + fp32 value
//   (12 bytes with fp64 values) -- no more than the CSR.
// Kernel (inside the persistent loop, loop_core.cuh): for each block the CTA
// TMA-copies x[block] (W doubles) into a double-buffered shared tile, warps
// stream their (slab, block, warp) entries with coalesced loads, gather x from
// shared memory, and fold each 32-entry chunk with a segmented warp scan into
// their own rows' shared accumulators (no atomics, deterministic order).
// L2->SM traffic per half: the entry stream + P copies of x instead of one
// random 32-byte sector per entry.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "loop_core.cuh"

namespace spk {

namespace {

constexpr int kNW = loopcore::kBlock / 32;  // warps per CTA (16)
constexpr int kMaxW = 16384;                // block width cap (col_local < 2^16)

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
// Bounded wait: returns false after ~2^24 polls (a lost transaction must not
// hang the GPU; the caller records a fault and the host raises it).
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

}  // namespace

namespace {

template <class VT>
struct BlockedOp {
  BlockedHalf L[2];
  int64_t n;
  int acc_rows;  // shared accumulator capacity (max rows of a slab)
  int W;         // shared tile width (max over halves)
  unsigned int* fault;  // set when a TMA transaction never completed

  static size_t smem_bytes(int W, int acc_rows) { return (size_t)2 * W * 8 + (size_t)acc_rows * 8 + 64; }
  size_t smem_bytes() const { return smem_bytes(W, acc_rows); }

  template <int ROLE, bool LOG, bool DET>
  __device__ void half(const double* x, const double* wgt, const double* old, double* out, unsigned char* ne,
                       int* dyn, double exponent, int policy, int t, unsigned long long* flag, double* absdiff,
                       double& err, long long& masks) const {
    extern __shared__ __align__(128) unsigned char dsm[];
    double* xb0 = reinterpret_cast<double*>(dsm);
    double* xb1 = xb0 + W;
    double* acc = xb1 + W;
    uint64_t* bar = reinterpret_cast<uint64_t*>(acc + acc_rows);
    const BlockedHalf& H = L[ROLE];
    const int p = blockIdx.x;
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const VT* val = static_cast<const VT*>(H.val);
    const int r0 = H.slab_row0[p];
    const int nrows = H.slab_row0[p + 1] - r0;

    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      fence_mbar_init();
    }
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) acc[r] = 0.0;
    __syncthreads();

    auto issue = [&](int b) {
      const int64_t c0 = (int64_t)b * H.W;
      const int64_t cnt = min((int64_t)H.W, H.n_in - c0);
      const uint32_t bytes = (uint32_t)(((cnt * 8) + 15) & ~int64_t(15));
      uint64_t* br = &bar[b & 1];
      mbar_arrive_expect_tx(br, bytes);
      bulk_copy_g2s((b & 1) ? xb1 : xb0, x + c0, bytes, br);
    };
    if (threadIdx.x == 0) {
      fence_proxy_async();  // x was written by generic stores before the grid barrier
      issue(0);
      if (H.B > 1) issue(1);
    }
    const int wrow0 = H.warp_row0[p * (kNW + 1) + w];
    (void)wrow0;
    for (int b = 0; b < H.B; ++b) {
      const double* xs = (b & 1) ? xb1 : xb0;
      if (!mbar_wait(&bar[b & 1], (uint32_t)((b >> 1) & 1))) atomicExch(fault, 1u);
      const long long beg = H.off[((int64_t)p * H.B + b) * kNW + w];
      const long long end = H.off[((int64_t)p * H.B + b) * kNW + w + 1];
      for (long long c = beg; c < end; c += 128) {
        uint32_t pk[4];
        double pr[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const long long e = c + lane + 32 * k;
          pk[k] = e < end ? __ldcs(H.packed + e) : 0xffffffffu;
          pr[k] = e < end ? (double)__ldcs(val + e) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (c + 32 * k >= end) break;  // warp-uniform
          const uint32_t rl = pk[k] >> 16;
          double s = pk[k] == 0xffffffffu ? 0.0 : pr[k] * xs[pk[k] & 0xffffu];
          // segmented inclusive scan over equal rl (rows ascend inside the chunk)
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const double so = __shfl_up_sync(0xffffffffu, s, d);
            const uint32_t ro = __shfl_up_sync(0xffffffffu, rl, d);
            if (lane >= d && ro == rl) s += so;
          }
          const uint32_t rn = __shfl_down_sync(0xffffffffu, rl, 1);
          const bool tail = (lane == 31) || (rn != rl);
          if (tail && pk[k] != 0xffffffffu) acc[rl] += s;
        }
      }
      __syncthreads();  // every warp is done with this tile
      if (threadIdx.x == 0 && b + 2 < H.B) issue(b + 2);
    }
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

__global__ void key_kernel(const long long* ptr, const uint32_t* idx, int64_t n_out, const int* slab_of,
                           const unsigned char* warp_of, int W, int B, uint32_t* keys) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_out; i += nw) {
    const uint32_t base = (uint32_t)slab_of[i] * (uint32_t)B;
    const uint32_t wv = warp_of[i];
    for (long long q = ptr[i] + lane; q < ptr[i + 1]; q += 32)
      keys[q] = (base + idx[q] / (uint32_t)W) * kNW + wv;
  }
}

template <class VT>
__global__ void pack_kernel(const uint32_t* perm, const long long* ptr, const uint32_t* idx, const VT* val,
                            const uint32_t* rows_of_pos, const int* slab_row0_of_row, int W, int64_t m,
                            uint32_t* packed, VT* vout) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t src = perm[q];
    const uint32_t i = rows_of_pos[src];
    const uint32_t rl = i - (uint32_t)slab_row0_of_row[i];
    const uint32_t cl = idx[src] % (uint32_t)W;
    packed[q] = (rl << 16) | cl;
    vout[q] = val[src];
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

// Build one half's layout from (ptr, idx, val): P slabs balanced by entries.
// Returns false when the shape does not fit (rows per slab >= 2^16).
bool build_blocked(spk_ctx* ctx, int P, int64_t n_out, int64_t n_in, int64_t m, const DBuf& ptr_d, const DBuf& idx_d,
                   const DBuf& val_d, int vbytes, size_t smem_budget, BlockedHost& out) {
  std::vector<long long> ptr(n_out + 1);
  download(ctx, ptr.data(), ptr_d, sizeof(long long) * (n_out + 1));
  // slab cut points: first row whose prefix reaches k*m/P
  std::vector<int> slab_row0(P + 1);
  slab_row0[0] = 0;
  for (int k = 1; k < P; ++k) {
    const long long target = (long long)((double)m * k / P);
    int r = (int)(std::lower_bound(ptr.begin(), ptr.end(), target) - ptr.begin());
    r = std::max(r, slab_row0[k - 1]);
    // also cap by rows so that no slab is far longer than n/P in rows
    slab_row0[k] = std::min<int64_t>(r, n_out);
  }
  slab_row0[P] = (int)n_out;
  int max_rows = 0;
  for (int k = 0; k < P; ++k) max_rows = std::max(max_rows, slab_row0[k + 1] - slab_row0[k]);
  if (max_rows >= 65536) return false;
  // shared tile width from the budget: 2 tiles of W doubles + accumulators
  const size_t acc_bytes = (size_t)max_rows * 8 + 64;
  if (smem_budget <= acc_bytes + 2 * 16 * 8) return false;
  int W = kMaxW;
  while (W > 16 && ((size_t)2 * W * 8 + acc_bytes > smem_budget || W > ctx->blocked_max_w)) W >>= 1;
  if ((int64_t)W > n_in) W = (int)std::max<int64_t>(16, ((n_in + 15) / 16) * 16);
  const int B = (int)((n_in + W - 1) / W);
  // warp cut points inside each slab (balanced by entries)
  std::vector<int> warp_row0((size_t)P * (kNW + 1));
  std::vector<int> slab_of(n_out);
  std::vector<unsigned char> warp_of(n_out);
  for (int k = 0; k < P; ++k) {
    const int a = slab_row0[k], z = slab_row0[k + 1];
    const long long e0 = ptr[a], e1 = ptr[z];
    int prev = a;
    warp_row0[(size_t)k * (kNW + 1)] = 0;
    for (int wv = 1; wv < kNW; ++wv) {
      const long long target = e0 + (long long)((double)(e1 - e0) * wv / kNW);
      int r = (int)(std::lower_bound(ptr.begin() + a, ptr.begin() + z, target) - ptr.begin());
      r = std::max(r, prev);
      warp_row0[(size_t)k * (kNW + 1) + wv] = r - a;
      prev = r;
    }
    warp_row0[(size_t)k * (kNW + 1) + kNW] = z - a;
    for (int wv = 0; wv < kNW; ++wv)
      for (int r = a + warp_row0[(size_t)k * (kNW + 1) + wv]; r < a + warp_row0[(size_t)k * (kNW + 1) + wv + 1]; ++r) {
        slab_of[r] = k;
        warp_of[r] = (unsigned char)wv;
      }
  }
  std::vector<int> slab_row0_of_row(n_out);
  for (int64_t r = 0; r < n_out; ++r) slab_row0_of_row[r] = slab_row0[slab_of[r]];

  cudaStream_t s = ctx->stream;
  DBuf d_slab_of, d_warp_of, d_s0r;
  upload(ctx, d_slab_of, slab_of.data(), sizeof(int) * n_out);
  upload(ctx, d_warp_of, warp_of.data(), n_out);
  upload(ctx, d_s0r, slab_row0_of_row.data(), sizeof(int) * n_out);
  upload(ctx, out.slab_row0, slab_row0.data(), sizeof(int) * (P + 1));
  upload(ctx, out.warp_row0, warp_row0.data(), sizeof(int) * warp_row0.size());
  const int64_t nkeys = (int64_t)P * B * kNW;
  if (nkeys >= (1LL << 32)) return false;
  const int64_t mm = std::max<int64_t>(m, 1);
  DBuf keys(sizeof(uint32_t) * mm), keys_s(sizeof(uint32_t) * mm), iota(sizeof(uint32_t) * mm),
      perm(sizeof(uint32_t) * mm), rows(sizeof(uint32_t) * mm), hist(sizeof(unsigned long long) * (nkeys + 1));
  out.off.alloc(sizeof(long long) * (nkeys + 1));
  out.packed.alloc(sizeof(uint32_t) * mm);
  out.val.alloc((size_t)vbytes * mm);
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
  SPK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<uint32_t>(), keys_s.as<uint32_t>(), iota.as<uint32_t>(),
                                           perm.as<uint32_t>(), (int)m, 0, end_bit, s));
  ctx->scratch.ensure(tb);
  SPK_CUDA(cub::DeviceRadixSort::SortPairs(ctx->scratch.p, tb, keys.as<uint32_t>(), keys_s.as<uint32_t>(),
                                           iota.as<uint32_t>(), perm.as<uint32_t>(), (int)m, 0, end_bit, s));
  SPK_CUDA(cudaMemsetAsync(out.off.p, 0, sizeof(long long), s));
  SPK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, hist.as<unsigned long long>(),
                                         out.off.as<unsigned long long>() + 1, (int)nkeys, s));
  ctx->scratch.ensure(tb);
  SPK_CUDA(cub::DeviceScan::InclusiveSum(ctx->scratch.p, tb, hist.as<unsigned long long>(),
                                         out.off.as<unsigned long long>() + 1, (int)nkeys, s));
  if (vbytes == 4)
    pack_kernel<float><<<grid_cap(ctx, m), 256, 0, s>>>(perm.as<uint32_t>(), ptr_d.as<long long>(),
                                                         idx_d.as<uint32_t>(), val_d.as<float>(), rows.as<uint32_t>(),
                                                         d_s0r.as<int>(), W, m, out.packed.as<uint32_t>(),
                                                         out.val.as<float>());
  else
    pack_kernel<double><<<grid_cap(ctx, m), 256, 0, s>>>(perm.as<uint32_t>(), ptr_d.as<long long>(),
                                                          idx_d.as<uint32_t>(), val_d.as<double>(), rows.as<uint32_t>(),
                                                          d_s0r.as<int>(), W, m, out.packed.as<uint32_t>(),
                                                          out.val.as<double>());
  ctx->launches += 3;
  SPK_CUDA(cudaGetLastError());
  SPK_CUDA(cudaStreamSynchronize(s));
  out.max_rows = max_rows;
  out.h.P = P;
  out.h.B = B;
  out.h.W = W;
  out.h.n_out = n_out;
  out.h.n_in = n_in;
  out.h.slab_row0 = out.slab_row0.as<int>();
  out.h.warp_row0 = out.warp_row0.as<int>();
  out.h.off = out.off.as<long long>();
  out.h.packed = out.packed.as<uint32_t>();
  out.h.val = out.val.p;
  return true;
}

// Runs the persistent loop with the blocked operator; returns false when the
// layout cannot be used (caller falls back to the CSR operator).
template <class VT>
bool run_blocked_t(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy,
                   LoopState& st, LoopOut& out) {
  const int64_t n = sk->n;
  if (!sk->blocked_tried) {
    sk->blocked_tried = true;
    int per_sm = 0;
    // one CTA per SM; the budget leaves room for the kernel's static shared memory
    const size_t budget = 200 * 1024;
    (void)per_sm;
    const int P = ctx->num_sms;
    auto R = std::make_unique<BlockedHost>(), C = std::make_unique<BlockedHost>();
    const int vb = sk->value_type == SPK_VALUES_F32 ? 4 : 8;
    if (build_blocked(ctx, P, n, n, sk->nnz, sk->row_ptr, sk->col_idx, sk->values, vb, budget, *R) &&
        build_blocked(ctx, P, n, n, sk->nnz, sk->col_ptr, sk->row_idx, sk->values_t, vb, budget, *C)) {
      sk->blk_rows = std::move(R);
      sk->blk_cols = std::move(C);
    }
  }
  if (!sk->blk_rows) return false;
  BlockedOp<VT> op;
  op.L[0] = sk->blk_rows->h;
  op.L[1] = sk->blk_cols->h;
  op.n = n;
  op.acc_rows = std::max(sk->blk_rows->max_rows, sk->blk_cols->max_rows);
  op.W = std::max(op.L[0].W, op.L[1].W);
  LoopWs& W = sk->ws;
  W.scalar.ensure(sizeof(unsigned int));
  SPK_CUDA(cudaMemsetAsync(W.scalar.p, 0, sizeof(unsigned int), ctx->stream));
  op.fault = W.scalar.as<unsigned int>();
  W.row_ne.ensure(n);
  W.col_ne.ensure(n);
  SPK_CUDA(cudaMemcpyAsync(W.row_ne.p, sk->cov_row.p, n, cudaMemcpyDeviceToDevice, ctx->stream));
  SPK_CUDA(cudaMemcpyAsync(W.col_ne.p, sk->cov_col.p, n, cudaMemcpyDeviceToDevice, ctx->stream));
  loopcore::run_core<false>(ctx, op, n, W, sk->cov_empty_rows, sk->cov_empty_cols, cfg, exponent, policy, st,
                            /*useful_blocks=*/op.L[0].P, out, /*exact_grid=*/op.L[0].P, op.smem_bytes());
  unsigned int fault = 0;
  download(ctx, &fault, W.scalar, sizeof fault);
  if (fault) fail_device("blocked loop: TMA tile never arrived", cudaErrorLaunchTimeout);
  return true;
}

bool run_blocked(spk_ctx* ctx, spk_sketch* sk, const spk_solver_cfg& cfg, double exponent, int policy, LoopState& st,
                 LoopOut& out) {
  if (sk->value_type == SPK_VALUES_F32) return run_blocked_t<float>(ctx, sk, cfg, exponent, policy, st, out);
  return run_blocked_t<double>(ctx, sk, cfg, exponent, policy, st, out);
}

}  // namespace spk
