// Microbenchmark probe (not product code): random 4-B gathers into windows of
// various sizes, alone and mixed with a sequential stream, to see how much of
// the 126 MB L2 a random-gather working set can actually use on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t hsh(uint64_t x){ x^=x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return (uint32_t)x; }
__global__ void k_gather(const int* __restrict__ t, uint32_t n_win, size_t n, int* out){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st=(size_t)gridDim.x*blockDim.x;
  int acc=0;
  for(; i<n; i+=st){ uint32_t j = hsh(i) % n_win; acc += __ldcg(t+j); }
  if(acc==0x12345) out[0]=acc;
}
// each step: one 16-B streamed load + G gathers into the window
template<int G>
__global__ void k_mix(const int4* __restrict__ s, size_t n4, const int* __restrict__ t, uint32_t n_win, int* out){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st=(size_t)gridDim.x*blockDim.x;
  int acc=0;
  for(; i<n4; i+=st){ int4 v = __ldcs(s+i); acc ^= v.x;
#pragma unroll
    for(int g=0; g<G; ++g){ uint32_t j = hsh(i*G+g) % n_win; acc += __ldcg(t+j); } }
  if(acc==0x12345) out[0]=acc;
}
int main(){
  int dev; CK(cudaGetDevice(&dev)); cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  printf("dev %s SMs %d L2 %d MB persistingL2max %d MB\n", p.name, p.multiProcessorCount, p.l2CacheSize>>20, p.persistingL2CacheMaxSize>>20);
  size_t big = (size_t)12<<30; char* buf; CK(cudaMalloc(&buf, big)); CK(cudaMemset(buf, 1, big));
  int* out; CK(cudaMalloc(&out, 4));
  int* tab = (int*)(buf + ((size_t)8<<30));   // window region (up to 4 GB)
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int G = p.multiProcessorCount*4;
  size_t ng = (size_t)1<<30;
  double mbs[] = {4, 16, 25.6, 40, 64, 96, 128, 256, 1024};
  for(double mb: mbs){ uint32_t w = (uint32_t)(mb*1e6/4);
    for(int r=0;r<2;r++){ cudaEventRecord(e0); k_gather<<<G,512>>>(tab, w, ng, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
    if(r) printf("gather window %7.1f MB: %8.3f ms for 2^30 -> %.3g gathers/s\n", mb, ms, ng/ms*1e3);} }
  size_t n4 = ((size_t)8<<30)/16;
  for(double mb: mbs){ uint32_t w = (uint32_t)(mb*1e6/4);
    for(int r=0;r<2;r++){ cudaEventRecord(e0); k_mix<4><<<G,512>>>((const int4*)buf, n4, tab, w, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
    if(r) printf("mix stream 8GB + 4 gathers/16B, window %7.1f MB: %8.3f ms -> stream %.0f GB/s, %.3g gathers/s\n", mb, ms, (8.0*(1<<30))/ms/1e6, n4*4.0/ms*1e3);} }
  CK(cudaDeviceSynchronize());
  return 0;
}
