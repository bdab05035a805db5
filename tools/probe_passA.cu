// Probe (not product code): pass-A replica on the real graph with L2 policy variants.
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t pol_last(){ uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;":"=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_first(){ uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;":"=l"(p)); return p; }
__device__ __forceinline__ int ld_hint(const int* p, uint64_t pol){ int r; asm volatile("ld.global.L2::cache_hint.b32 %0, [%1], %2;":"=r"(r):"l"(p),"l"(pol)); return r; }
__device__ __forceinline__ int4 ld4_hint(const void* p, uint64_t pol){ int4 r; asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;":"=r"(r.x),"=r"(r.y),"=r"(r.z),"=r"(r.w):"l"(p),"l"(pol)); return r; }
template <int M>
__global__ void k_passA(const int32_t* __restrict__ nbr, const float* __restrict__ dist, int k, int64_t n,
                        const int32_t* __restrict__ comp, int* out) {
  int acc = 0;
  const uint64_t pl = pol_last(), pf = pol_first();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    int4 j4, w4;
    if (M & 2) { j4 = ld4_hint(nbr + r * k, pf); w4 = ld4_hint(dist + r * k, pf); }
    else { j4 = __ldcs(reinterpret_cast<const int4*>(nbr + r * k)); w4 = __ldcs(reinterpret_cast<const int4*>(dist + r * k)); }
    if (M & 1) acc += ld_hint(comp + j4.x, pl) + ld_hint(comp + j4.y, pl) + ld_hint(comp + j4.z, pl) + ld_hint(comp + j4.w, pl);
    else acc += __ldcg(comp + j4.x) + __ldcg(comp + j4.y) + __ldcg(comp + j4.z) + __ldcg(comp + j4.w);
    acc += w4.x;
  }
  if (acc == 0x1234567) out[0] = acc;
}
extern "C" float probe_passA(const int32_t* nbr, const float* dist, int k, int64_t n, const int32_t* comp, int mode, int carve_mb, int window) {
  int* out; cudaMalloc(&out, 4);
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)carve_mb << 20);
  cudaStream_t st; cudaStreamCreate(&st);
  if (window) {
    cudaStreamAttrValue a = {};
    a.accessPolicyWindow.base_ptr = (void*)comp;
    a.accessPolicyWindow.num_bytes = (size_t)n * 4;
    a.accessPolicyWindow.hitRatio = (float)((double)((size_t)carve_mb << 20) / ((double)n * 4));
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
  }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto launch = [&]() {
    if (mode == 0) k_passA<0><<<1184, 256, 0, st>>>(nbr, dist, k, n, comp, out);
    else if (mode == 1) k_passA<1><<<1184, 256, 0, st>>>(nbr, dist, k, n, comp, out);
    else if (mode == 2) k_passA<2><<<1184, 256, 0, st>>>(nbr, dist, k, n, comp, out);
    else k_passA<3><<<1184, 256, 0, st>>>(nbr, dist, k, n, comp, out);
  };
  launch();
  cudaEventRecord(a, st); launch(); cudaEventRecord(b, st); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaCtxResetPersistingL2Cache();
  cudaStreamDestroy(st); cudaFree(out); return ms;
}
