// Probe (not product code): replay the k_offer_warp access pattern on the real
// graph, adding one ingredient at a time.
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_gather_rows(const int32_t* __restrict__ nbr, const float* __restrict__ dist, int k, int64_t r0,
                              int64_t r1, int stride, const int32_t* __restrict__ comp, int mode,
                              unsigned long long* __restrict__ Kc, uint16_t* __restrict__ head,
                              unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
  unsigned acc = 0;
  for (int64_t r = r0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32 * stride; r < r1; r += nw * stride) {
    int cv = (mode >= 3) ? __ldcg(comp + r) : 0;
    int h = (mode >= 4) ? head[r] : 0;
    unsigned long long best = ~0ull;
    for (int c = (h & ~31) + lane; c < k; c += 32) {
      int J = __ldcs(nbr + r * k + c);
      float w = (mode >= 2) ? __ldcs(dist + r * k + c) : 0.f;
      int cj = __ldcg(comp + J);
      acc += cj;
      if (mode >= 5 && cj != cv) best = min(best, ((unsigned long long)__float_as_uint(w) << 32) | (unsigned)J);
    }
    if (mode >= 5) {
      for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (lane == 0 && best != ~0ull) atomicMin(Kc + cv, best);
    }
    if (mode >= 4 && lane == 0) head[r] = (uint16_t)k;
  }
  if (acc == 0x12345) atomicAdd(out, 1ull);
}
extern "C" float probe_gather(const int32_t* nbr, const float* dist, int k, int64_t r0, int64_t r1, int stride,
                              const int32_t* comp, int mode, unsigned long long* Kc, uint16_t* head) {
  unsigned long long* out; cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_gather_rows<<<148 * 8, 256>>>(nbr, dist, k, r0, r1, stride, comp, mode, Kc, head, out);
  cudaEventRecord(a);
  k_gather_rows<<<148 * 8, 256>>>(nbr, dist, k, r0, r1, stride, comp, mode, Kc, head, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); cudaFree(out); return ms;
}
