// Probe (not product code): 4 random gathers per "row" into a W-byte window while
// streaming 2 x 16 B per row from a huge buffer (the pass-A pattern), with L2
// eviction-priority variants.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint64_t x){ x^=x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return (uint32_t)x; }
__device__ __forceinline__ uint64_t pol_last(){ uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;":"=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_first(){ uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;":"=l"(p)); return p; }
__device__ __forceinline__ int ld_hint(const int* p, uint64_t pol){ int r; asm volatile("ld.global.L2::cache_hint.b32 %0, [%1], %2;":"=r"(r):"l"(p),"l"(pol)); return r; }
__device__ __forceinline__ int4 ld4_hint(const int4* p, uint64_t pol){ int4 r; asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;":"=r"(r.x),"=r"(r.y),"=r"(r.z),"=r"(r.w):"l"(p),"l"(pol)); return r; }
template<int MODE>
__global__ void k(const int* __restrict__ win, uint32_t wn, const int4* __restrict__ A, const int4* __restrict__ B, size_t rows, int* out){
  uint64_t pl = pol_last(), pf = pol_first();
  int acc=0;
  for(size_t r = blockIdx.x*(size_t)blockDim.x + threadIdx.x; r < rows; r += (size_t)gridDim.x*blockDim.x){
    int4 a, b;
    if (MODE >= 2) { a = ld4_hint(A + r*25, pf); b = ld4_hint(B + r*25, pf); }
    else { a = __ldcs(A + r*25); b = __ldcs(B + r*25); }
    int js[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int j=0;j<4;++j){ uint32_t J = hsh(r*4+j+js[j]*0) % wn; acc += (MODE>=1) ? ld_hint(win + J, pl) : __ldcg(win + J); }
    acc ^= b.x;
  }
  if(acc==0x1234567) out[0]=acc;
}
int main(){
  size_t rows = 64000000; size_t bytes = rows*400;
  int4 *A,*B; cudaMalloc(&A, bytes); cudaMalloc(&B, bytes); cudaMemset(A,0,bytes); cudaMemset(B,0,bytes);
  int* win; cudaMalloc(&win, 256<<20); cudaMemset(win,0,256<<20); int* out; cudaMalloc(&out,4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int carve : {0, 64, 96}) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)carve<<20);
    size_t got=0; cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
    for (uint32_t wn : {6400000u, 16000000u}) for (int mode=0; mode<3; ++mode) for (int r=0;r<2;++r){
      cudaEventRecord(e0);
      if(mode==0) k<0><<<1184,256>>>(win,wn,A,B,rows,out); else if(mode==1) k<1><<<1184,256>>>(win,wn,A,B,rows,out); else k<2><<<1184,256>>>(win,wn,A,B,rows,out);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
      if(r) printf("carve %zu MB window %.1f MB mode %d (0 plain,1 gather evict_last,2 +stream evict_first): %.2f ms  %.3g gathers/s\n", got>>20, wn*4/1e6, mode, ms, rows*4/ms*1e3);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
