// Peak MUFU.EX2 and FFMA throughput per SM on this B200 (the
// dense on-the-fly comparator's roofline denominator is measured on the box).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sfu_fma_peak sfu_fma_peak.cu && ./sfu_fma_peak
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void spin(float* out, int iters, float seed) {
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = seed + 0.001f * (threadIdx.x + k);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[k]));
      else v[k] = fmaf(v[k], 0.999f, 0.0001f);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  if (s == 12345.f) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz (max)
  float* out;
  cudaMalloc(&out, 4);
  const int blocks = sms * 4, threads = 512, iters = 1 << 14;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int op = 0; op < 2; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (op == 0) spin<0><<<blocks, threads>>>(out, iters, -0.5f);
      else spin<1><<<blocks, threads>>>(out, iters, 0.5f);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)blocks * threads * iters * 8;
      if (rep == 1)
        std::printf("%s: %.3e ops/s = %.1f per clk per SM at the %d MHz max clock\n", op == 0 ? "MUFU.EX2" : "FFMA",
                    ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
