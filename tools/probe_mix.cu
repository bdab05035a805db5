// Probe (not product code): random 4-B gathers into a W-byte window while the
// same kernel streams a large buffer; does the stream evict the window from L2?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint64_t x){ x^=x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return (uint32_t)x; }
template<int MODE>
__global__ void k_mix(const int* __restrict__ win, uint32_t wn, const int4* __restrict__ stream, size_t sn, size_t iters, int ratio, int* out){
  size_t t = blockIdx.x*(size_t)blockDim.x + threadIdx.x, T=(size_t)gridDim.x*blockDim.x;
  int acc=0;
  for(size_t it=t; it<iters; it+=T){
    if(ratio){ // one 16-B stream load per `ratio` gathers
      if((it % ratio)==0){ const int4* p = stream + ((it/ratio) % sn); int4 v;
        if(MODE==0) v = __ldg(p); else if(MODE==1) v = __ldcs(p); else { asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];":"=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w):"l"(p)); }
        acc ^= v.x; }
    }
    acc += __ldcg(win + (hsh(it) % wn));
  }
  if(acc==0x1234567) out[0]=acc;
}
int main(){
  size_t sbytes=(size_t)16<<30; int4* st; cudaMalloc(&st, sbytes); cudaMemset(st,1,sbytes);
  int* win; cudaMalloc(&win, 512<<20); cudaMemset(win,0,512<<20); int* out; cudaMalloc(&out,4);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  size_t iters=(size_t)1<<30; int G=148*16;
  uint32_t wins[]={6400000u, 16000000u, 64000000u};
  for(uint32_t w: wins) for(int ratio: {0, 8, 2}) for(int mode=0; mode<3; ++mode){
    if(ratio==0 && mode>0) continue;
    for(int r=0;r<2;r++){ cudaEventRecord(a);
      if(mode==0) k_mix<0><<<G,256>>>(win,w,st,sbytes/16,iters,ratio,out);
      else if(mode==1) k_mix<1><<<G,256>>>(win,w,st,sbytes/16,iters,ratio,out);
      else k_mix<2><<<G,256>>>(win,w,st,sbytes/16,iters,ratio,out);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
      if(r) printf("window %.1f MB  stream 1/%d  mode %d (0 ldg,1 ldcs,2 nc.noalloc.evict_first): %.2f ms  %.3g gathers/s  stream %.0f GB/s\n", w*4/1e6, ratio, mode, ms, iters/ms*1e3, ratio? (double)iters/ratio*16/ms/1e6 : 0.0);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
