// Microbenchmark: 1-D TMA bulk-copy (cp.async.bulk) streaming throughput on
// B200 as a function of chunk size and pipeline depth, vs plain coalesced
// LDG streaming. One CTA per SM streams a disjoint slice of a 2 GB buffer.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
__device__ __forceinline__ void minit(uint64_t* b,uint32_t c){asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"::"r"(sa(b)),"r"(c):"memory");}
__device__ __forceinline__ void mexp(uint64_t* b,uint32_t n){asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(sa(b)),"r"(n):"memory");}
__device__ __forceinline__ void marr(uint64_t* b){asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"::"r"(sa(b)):"memory");}
__device__ __forceinline__ void mwait(uint64_t* b,uint32_t ph){asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}"::"r"(sa(b)),"r"(ph):"memory");}
__device__ __forceinline__ void bulk(void* d,const void* s,uint32_t n,uint64_t* b){asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"::"r"(sa(d)),"l"(s),"r"(n),"r"(sa(b)):"memory");}
extern __shared__ __align__(128) unsigned char sm[];
// consumers: all warps read the stage (sum) then release
__global__ void tma_stream(const unsigned char* src, size_t slice, int chunk, int S, int ncopies, double* out){
  uint64_t* full=(uint64_t*)(sm + (size_t)S*chunk); uint64_t* empty=full+S;
  const unsigned char* base=src + blockIdx.x*slice;
  int nchunks = (int)(slice/chunk);
  if(threadIdx.x==0){for(int s=0;s<S;++s){minit(&full[s],1);minit(&empty[s],blockDim.x/32);} asm volatile("fence.mbarrier_init.release.cluster;");}
  __syncthreads();
  auto issue=[&](int c){int s=c%S; mexp(&full[s],chunk); int part=chunk/ncopies; for(int k=0;k<ncopies;++k) bulk(sm+(size_t)s*chunk+k*part, base+(size_t)c*chunk+k*part, part,&full[s]);};
  if(threadIdx.x==0) for(int c=0;c<S&&c<nchunks;++c) issue(c);
  double acc=0; int lane=threadIdx.x&31;
  for(int c=0;c<nchunks;++c){int s=c%S; mwait(&full[s],(c/S)&1);
    const float* f=(const float*)(sm+(size_t)s*chunk);
    for(int i=threadIdx.x;i<chunk/4;i+=blockDim.x) acc+=f[i];
    __syncwarp(); if(lane==0) marr(&empty[s]);
    if(threadIdx.x==0 && c+S<nchunks){mwait(&empty[s],(c/S)&1); issue(c+S);} }
  if(acc==12345.0) out[0]=acc;
}
__global__ void ldg_stream(const float4* src, size_t n4, double* out){
  double acc=0; for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n4;i+=(size_t)gridDim.x*blockDim.x){float4 v=__ldcs(src+i); acc+=v.x+v.y+v.z+v.w;}
  if(acc==12345.0) out[0]=acc;
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  size_t bytes=(size_t)2<<30; unsigned char* buf; cudaMalloc(&buf,bytes); cudaMemset(buf,0,bytes); double* out; cudaMalloc(&out,8);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  size_t slice=(bytes/sms)&~(size_t)65535;
  for(int chunk: {4096,8192,16384,32768,65536}) for(int S: {2,4,6,8}) for(int nc: {1,4}){
    size_t smem=(size_t)S*chunk+2*S*8+16; if(smem>227*1024) continue;
    cudaFuncSetAttribute(tma_stream,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)smem);
    for(int threads: {256,512}){
      tma_stream<<<sms,threads,smem>>>(buf,slice,chunk,S,nc,out); cudaDeviceSynchronize();
      cudaEventRecord(a); for(int r=0;r<3;++r) tma_stream<<<sms,threads,smem>>>(buf,slice,chunk,S,nc,out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms,a,b); cudaError_t e=cudaGetLastError();
      printf("tma chunk=%6d S=%d copies=%d threads=%d : %7.1f GB/s %s\n",chunk,S,nc,threads, 3.0*slice*sms/(ms*1e6), e?cudaGetErrorString(e):"");
    }
  }
  for(int g: {1,2,4,8}){ ldg_stream<<<sms*g,512>>>((float4*)buf,bytes/16,out); cudaEventRecord(a); for(int r=0;r<3;++r) ldg_stream<<<sms*g,512>>>((float4*)buf,bytes/16,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b); printf("ldg grid=%d x sms: %7.1f GB/s\n",g,3.0*bytes/(ms*1e6)); }
  return 0;
}
