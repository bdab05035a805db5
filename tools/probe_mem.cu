// Microbenchmark probe (not product code): streaming read BW, random 4-B gather
// throughput from windows of various sizes, and random 64-bit atomicMin throughput.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__global__ void k_stream(const int4* __restrict__ a, size_t n4, int* out){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st = (size_t)gridDim.x*blockDim.x;
  int acc=0;
  for(; i<n4; i+=st){ int4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];":"=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w):"l"(a+i)); acc ^= v.x^v.y^v.z^v.w; }
  if(acc==0x12345) out[0]=acc;
}
__device__ __forceinline__ uint32_t hsh(uint64_t x){ x^=x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return (uint32_t)x; }
__global__ void k_gather(const int* __restrict__ t, uint32_t mask_n, size_t n, int* out){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st=(size_t)gridDim.x*blockDim.x;
  int acc=0;
  for(; i<n; i+=st){ uint32_t j = hsh(i) % mask_n; acc += __ldg(t+j); }
  if(acc==0x12345) out[0]=acc;
}
__global__ void k_atom(unsigned long long* t, uint32_t mask_n, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st=(size_t)gridDim.x*blockDim.x;
  for(; i<n; i+=st){ uint32_t j = hsh(i) % mask_n; atomicMin(t+j, (unsigned long long)hsh(i*7)); }
}
__global__ void k_atom_ret(unsigned long long* t, uint32_t mask_n, size_t n, int* out){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st=(size_t)gridDim.x*blockDim.x;
  unsigned long long acc=0;
  for(; i<n; i+=st){ uint32_t j = hsh(i) % mask_n; acc += atomicMin(t+j, (unsigned long long)hsh(i*7)); }
  if(acc==0x12345) out[0]=1;
}
int main(){
  int dev; CK(cudaGetDevice(&dev)); cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  printf("dev %s SMs %d L2 %d MB\n", p.name, p.multiProcessorCount, p.l2CacheSize>>20);
  size_t big = (size_t)8<<30; void* buf; CK(cudaMalloc(&buf, big)); CK(cudaMemset(buf, 1, big));
  int* out; CK(cudaMalloc(&out, 4));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int G = p.multiProcessorCount*8;
  for(int r=0;r<3;r++){ cudaEventRecord(e0); k_stream<<<G,512>>>((int4*)buf, big/16, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
    printf("stream read 8GB: %.3f ms  %.1f GB/s\n", ms, big/ms/1e6); }
  size_t ng = (size_t)1<<30;
  uint32_t wins[] = {1u<<18, 1u<<21, 1u<<23, 6400000u, 1u<<24, 1u<<26, 64000000u, 1u<<28};
  for(uint32_t w: wins){ for(int r=0;r<2;r++){ cudaEventRecord(e0); k_gather<<<G,512>>>((int*)buf, w, ng, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
    if(r) printf("gather window %u ints (%.1f MB): %.3f ms for 2^30 -> %.3g gathers/s\n", w, w*4/1e6, ms, ng/ms*1e3);} }
  size_t na = (size_t)1<<28;
  for(uint32_t w: wins){ for(int r=0;r<2;r++){ cudaEventRecord(e0); k_atom<<<G,512>>>((unsigned long long*)buf, w/2, na); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
    if(r) printf("red.min.u64 window %u (%.1f MB): %.3f ms for 2^28 -> %.3g atom/s\n", w/2, w*4/1e6, ms, na/ms*1e3);} }
  for(uint32_t w: wins){ for(int r=0;r<2;r++){ cudaEventRecord(e0); k_atom_ret<<<G,512>>>((unsigned long long*)buf, w/2, na, out); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
    if(r) printf("atom.min.u64(ret) window %u (%.1f MB): %.3f ms for 2^28 -> %.3g atom/s\n", w/2, w*4/1e6, ms, na/ms*1e3);} }
  CK(cudaDeviceSynchronize());
  return 0;
}
