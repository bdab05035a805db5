// Probe (not product code): 4 hash-random gathers per "row" into (a) a 25.6 MB
// window that moves every 6.4M rows, (b) a fixed 25.6 MB window; no stream.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint64_t x){ x^=x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return (uint32_t)x; }
template<int MOVING>
__global__ void kw(const int* __restrict__ comp, int64_t rows, int per, int* out){
  int acc=0;
  for(int64_t r = blockIdx.x*(int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x*blockDim.x){
    const int64_t base = MOVING ? (r / 6400000) * 6400000 : 0;
    for (int j = 0; j < per; ++j) acc += __ldcg(comp + base + hsh(r * 8 + j) % 6400000);
  }
  if(acc==0x1234567) out[0]=acc;
}
int main(){
  int* comp; cudaMalloc(&comp, 64000000*4); cudaMemset(comp, 0, 64000000*4); int* out; cudaMalloc(&out,4);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for (int per : {4, 32}) for (int mv = 0; mv < 2; ++mv) for (int it = 0; it < 2; ++it) {
    cudaEventRecord(a);
    if (mv) kw<1><<<1184,256>>>(comp, 64000000, per, out); else kw<0><<<1184,256>>>(comp, 64000000, per, out);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    if (it) printf("gathers/row %d moving %d: %.2f ms  %.3g gathers/s\n", per, mv, ms, 64e6*per/ms*1e3);
  }
  return 0;
}
