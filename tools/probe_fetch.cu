// Probe: DRAM fetch granularity of scattered 4-B loads (one per 400-B row, the
// k_core_mark / k_label pattern) under cudaLimitMaxL2FetchGranularity and load
// flavours.  Prints ms and effective bytes per load at HBM peak.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_probe(const float* __restrict__ d, int64_t rows, int k, int col, float eps, uint32_t* out) {
  const int64_t w1 = (rows + 31) >> 5;
  for (int64_t wd = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; wd < w1; wd += (int64_t)gridDim.x * blockDim.x) {
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t v = (wd << 5) + j;
      float x = 1e30f;
      if (v < rows) {
        const float* p = d + v * k + col;
        if (MODE == 0) x = __ldcs(p);
        else if (MODE == 1) x = __ldg(p);
        else if (MODE == 2) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(x) : "l"(p));
        else if (MODE == 3) asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(x) : "l"(p));
        else x = *(volatile const float*)p;
      }
      word |= (x <= eps ? 1u : 0u) << j;
    }
    out[wd] = word;
  }
}

int main() {
  const int64_t rows = 64000000; const int k = 100;
  float* d; uint32_t* out;
  cudaMalloc(&d, rows * k * 4); cudaMalloc(&out, rows / 8 + 64);
  cudaMemset(d, 0, rows * k * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int gran[4] = {0, 32, 64, 128};
  for (int gi = 0; gi < 4; ++gi) {
    if (gran[gi]) { cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran[gi]); if (e) printf("limit %d: %s\n", gran[gi], cudaGetErrorString(e)); }
    size_t cur = 0; cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity);
    for (int mode = 0; mode < 5; ++mode) {
      float best = 1e9;
      for (int it = 0; it < 4; ++it) {
        cudaEventRecord(a);
        switch (mode) {
          case 0: k_probe<0><<<296 * 4, 256>>>(d, rows, k, 49, 0.5f, out); break;
          case 1: k_probe<1><<<296 * 4, 256>>>(d, rows, k, 49, 0.5f, out); break;
          case 2: k_probe<2><<<296 * 4, 256>>>(d, rows, k, 49, 0.5f, out); break;
          case 3: k_probe<3><<<296 * 4, 256>>>(d, rows, k, 49, 0.5f, out); break;
          default: k_probe<4><<<296 * 4, 256>>>(d, rows, k, 49, 0.5f, out); break;
        }
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      printf("limit(set %d, now %zu) mode %d: %.3f ms  -> %.0f B/load at 6.5 TB/s\n", gran[gi], cur, mode, best,
             best * 1e-3 * 6.5e12 / rows);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
