// Microbenchmark: which lane groupings of a 64-bit shared load conflict on B200?
// 16 warps on one SM issue independent LDS.64 back to back; cycles per
// instruction = wavefronts per instruction (the shared data pipe moves one
// 128-byte wavefront per cycle). Pattern p gives lane l the fp64 slot idx(p, l).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds64_conflicts lds64_conflicts.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ double lds(uint32_t a) { double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory"); return v; }
__device__ __forceinline__ void sts(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" :: "r"(a), "d"(v)); }
__device__ int slot(int p, int l) {
  switch (p) {
    case 0: return l;                                   // 32 consecutive doubles: ideal (2 wavefronts)
    case 1: return (l & 15) + 32 * (l >> 4);            // halves 0-15 / 16-31 each cover the 16 bank pairs once
    case 2: return (l >> 1) + 16 * (l & 1) * 3;         // lanes 2i, 2i+1 share a bank pair: each half has 8 pairs twice
    case 3: return (l & 7) + 16 * (l >> 3);             // only 8 bank pairs used, 4 lanes each (one per quarter)
    case 4: return (l & 15) * 16;                       // all lanes in bank pair 0 (lanes l, l+16 same address)
    case 5: return ((l & 15) >> 1) + 16 * (l & 1) + 32 * (l >> 4) * 2;  // per half: 8 pairs twice (as 2, other lane order)
    case 6: return (l & 1) ? (l >> 1) + 16 : (l >> 1) + 64;  // even lanes pairs 0-15 once, odd lanes pairs 0-15 once
    case 7: return (l < 16) ? (l & 7) + 16 * (l >> 3) : 8 + (l & 7) + 16 * ((l >> 3) & 1) + 64;  // half 0 uses pairs 0-7 twice, half 1 pairs 8-15 twice
    case 8: return (l < 16) ? l : 16 + 16 * (l - 16);   // half 0 ideal, half 1 all in bank pair 0 (16-way)
    case 9: return (l % 3 == 0) ? l : l + 16 * 5;       // same bank pair as 0, other rows: no conflicts, scattered
  }
  return l;
}
template <bool STORE>
__global__ void k(int p, int iters, long long* out, double* sink) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const int l = threadIdx.x & 31;
  // every warp reads its own rows (same bank pattern): identical addresses across warps would be merged
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(sm) + 8u * (uint32_t)(slot(p, l) + 16 * (threadIdx.x >> 5));
  double acc = 0, accs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (STORE) sts(a + 1024u * u, acc); else accs[u & 7] += lds(a + 1024u * u);  // 8 chains: not DADD-latency bound
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  for (int u = 0; u < 8; ++u) acc += accs[u];
  if (acc == 1.2345) sink[0] = acc;
}
int main() {
  long long* out; double* sink; cudaMalloc(&out, 8); cudaMalloc(&sink, 8);
  const int iters = 2000, warps = 16;
  for (int st = 0; st < 2; ++st)
    for (int p = 0; p < 10; ++p) {
      if (st) k<true><<<1, 32 * warps, 32768>>>(p, iters, out, sink); else k<false><<<1, 32 * warps, 32768>>>(p, iters, out, sink);
      long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      printf("%s pattern %d: %.2f cycles per instruction %s\n", st ? "STS.64" : "LDS.64", p, (double)c / ((double)iters * 16 * warps), cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
