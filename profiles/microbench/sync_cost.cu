// sync_cost.cu -- microbenchmark: cost of one cluster barrier (CS = 2..16
// CTAs of 1024 threads), one __syncthreads, and one cooperative grid.sync
// (148 CTAs), each repeated 20000 times in one launch; prints us per barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_cost sync_cost.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void cluster_bar(int iters, int* sink) {
  for (int k = 0; k < iters; ++k)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = iters;
}
__global__ void cta_bar(int iters, int* sink) {
  for (int k = 0; k < iters; ++k) __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = iters;
}
__global__ void grid_bar(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  for (int k = 0; k < iters; ++k) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = iters;
}

template <class F>
float timed(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int* sink;
  cudaMalloc(&sink, 4);
  const int iters = 20000;
  for (int cs : {2, 4, 8, 16}) {
    cudaFuncSetAttribute(cluster_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cs);
    lc.blockDim = dim3(1024);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    float ms = timed([&] { cudaLaunchKernelEx(&lc, cluster_bar, iters, sink); });
    printf("cluster barrier CS=%2d: %.3f us\n", cs, 1e3 * ms / iters);
  }
  float ms = timed([&] { cta_bar<<<1, 1024>>>(iters, sink); });
  printf("__syncthreads (1024 threads): %.3f us\n", 1e3 * ms / iters);
  for (int g : {148, 296}) {
    void* args[] = {(void*)&iters, (void*)&sink};
    ms = timed([&] { cudaLaunchCooperativeKernel((void*)grid_bar, g, 512, args, 0, 0); });
    printf("grid.sync (%d CTAs x 512): %.3f us\n", g, 1e3 * ms / iters);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
