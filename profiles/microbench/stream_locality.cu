// Microbenchmark: how the shape of per-warp entry streams limits HBM read
// throughput on B200. One 512-thread CTA per SM, 15 streaming warps (as in
// the slab x block loop, blocked.cu), each with DEPTH "groups" in flight in
// registers; a group is one 16-byte load per lane from a key plane and one
// from a value plane.
//   layout 0: per-warp streams, key and value planes in separate arrays (512 B runs)
//   layout 1: per-warp streams, key|value interleaved per group (1 KB runs)
//   layout 2: CTA-interleaved: group g of warp w at ((g * NW + w) * 1 KB) (15 KB runs)
//   layout 3: as 2, but keys of all warps then values of all warps per step (2 x 7.5 KB runs)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_locality stream_locality.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int NW = 15;
__device__ __forceinline__ uint64_t pol_ef() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint4 ldg_s(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}
template <int LAYOUT, int DEPTH>
__global__ void __launch_bounds__(512, 1) stream_kernel(const unsigned char* buf, size_t cta_bytes, int ngroups, unsigned* out) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w >= NW) return;
  const unsigned char* base = buf + blockIdx.x * cta_bytes;
  const uint64_t pol = pol_ef();
  auto addr_k = [&](int g) -> const unsigned char* {
    if (LAYOUT == 0) return base + ((size_t)w * ngroups + g) * 512 + lane * 16;
    if (LAYOUT == 1) return base + ((size_t)w * ngroups + g) * 1024 + lane * 16;
    if (LAYOUT == 2) return base + ((size_t)g * NW + w) * 1024 + lane * 16;
    return base + ((size_t)g * 2 * NW + w) * 512 + lane * 16;
  };
  auto addr_v = [&](int g) -> const unsigned char* {
    if (LAYOUT == 0) return base + cta_bytes / 2 + ((size_t)w * ngroups + g) * 512 + lane * 16;
    if (LAYOUT == 1) return base + ((size_t)w * ngroups + g) * 1024 + 512 + lane * 16;
    if (LAYOUT == 2) return base + ((size_t)g * NW + w) * 1024 + 512 + lane * 16;
    return base + ((size_t)g * 2 * NW + NW + w) * 512 + lane * 16;
  };
  uint4 K[DEPTH], V[DEPTH];
#pragma unroll
  for (int d = 0; d < DEPTH; ++d) { K[d] = ldg_s(addr_k(d), pol); V[d] = ldg_s(addr_v(d), pol); }
  unsigned acc = 0;
  for (int g0 = 0; g0 < ngroups; g0 += DEPTH) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      const uint4 k = K[d], v = V[d];
      const int gn = min(g0 + d + DEPTH, ngroups - 1);
      K[d] = ldg_s(addr_k(gn), pol); V[d] = ldg_s(addr_v(gn), pol);
      acc += k.x ^ k.y ^ k.z ^ k.w ^ v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}
template <int LAYOUT, int DEPTH>
void run(const unsigned char* buf, size_t cta_bytes, int sms, unsigned* out) {
  const int ngroups = (int)(cta_bytes / (NW * 1024)) / DEPTH * DEPTH;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  stream_kernel<LAYOUT, DEPTH><<<sms, 512>>>(buf, cta_bytes, ngroups, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) stream_kernel<LAYOUT, DEPTH><<<sms, 512>>>(buf, cta_bytes, ngroups, out);
  cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  printf("layout %d depth %d: %7.1f GB/s %s\n", LAYOUT, DEPTH, 5.0 * ngroups * NW * 1024.0 * sms / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t bytes = (size_t)2 << 30; unsigned char* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  unsigned* out; cudaMalloc(&out, 8);
  const size_t cta_bytes = (bytes / sms) & ~(size_t)(65535);
  run<0, 2>(buf, cta_bytes, sms, out); run<0, 3>(buf, cta_bytes, sms, out); run<0, 4>(buf, cta_bytes, sms, out); run<0, 6>(buf, cta_bytes, sms, out);
  run<1, 2>(buf, cta_bytes, sms, out); run<1, 3>(buf, cta_bytes, sms, out); run<1, 4>(buf, cta_bytes, sms, out); run<1, 6>(buf, cta_bytes, sms, out);
  run<2, 2>(buf, cta_bytes, sms, out); run<2, 3>(buf, cta_bytes, sms, out); run<2, 4>(buf, cta_bytes, sms, out); run<2, 6>(buf, cta_bytes, sms, out);
  run<3, 3>(buf, cta_bytes, sms, out); run<3, 4>(buf, cta_bytes, sms, out);
  return 0;
}
