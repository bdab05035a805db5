// Probe (not product code): the access pattern of one early light round at C4
// (64M live rows in row order; per row: an 8-B record, one 32-B ELL chunk,
// comp[v], G random comp[J] gathers with J uniform inside the row's cluster
// window of 6.4M ids, and one offer into a per-component slot of a random
// component of the same cluster), with pieces switched off one at a time, to
// see which part of the working set defeats the L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_round tools/probe_round.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t hsh(uint64_t x){ x^=x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return (uint32_t)x; }
__device__ __forceinline__ void ld256cs(const int4* p, int4& a, int4& b) {
  asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p));
}
__device__ __forceinline__ uint64_t pol_last(){ uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;":"=l"(p)); return p; }
__device__ __forceinline__ int ld_last(const int* p, uint64_t pol){ int r; asm volatile("ld.global.L2::cache_hint.b32 %0, [%1], %2;":"=r"(r):"l"(p),"l"(pol)); return r; }

struct P { int ell, compv, G, kb, last; uint32_t win, cwin; };
// rows in order: block grabs chunks of 1024 from a cursor (as the product kernels)
__global__ void __launch_bounds__(256) k_round(const int2* __restrict__ rec, const int4* __restrict__ LE,
    const int* __restrict__ comp, unsigned long long* __restrict__ Kc, ulonglong2* KB, size_t rows, P p,
    unsigned* grab, int* out) {
  __shared__ unsigned s_chunk;
  uint64_t pl = pol_last();
  int acc = 0;
  for (;;) {
    if (threadIdx.x == 0) s_chunk = atomicAdd(grab, 1u);
    __syncthreads();
    size_t base = (size_t)s_chunk * 1024;
    __syncthreads();
    if (base >= rows) break;
    for (int t = 0; t < 1024; t += 256) {
      size_t s = base + t + threadIdx.x;
      if (s >= rows) continue;
      int2 r = __ldcs(rec + s);
      int v = r.x;
      uint32_t cl = (uint32_t)(v / p.win);
      int4 a = make_int4(0,0,0,0), b = a;
      if (p.ell) ld256cs(LE + (size_t)v * 8, a, b);
      int cv = p.compv ? __ldcg(comp + v) : v;
      int js[4] = {a.x, a.z, b.x, b.z};
      int best = 0x7fffffff;
      for (int j = 0; j < p.G; ++j) {
        uint32_t J = cl * p.win + (hsh((uint64_t)s * 8 + j) + (uint32_t)js[j & 3]) % p.win;
        int c = p.last ? ld_last(comp + J, pl) : __ldcg(comp + J);
        if (c != cv) best = min(best, c);
      }
      acc ^= best;
      if (p.kb) {
        uint32_t cc = cl * p.cwin + hsh((uint64_t)v * 3 + 1) % p.cwin;
        unsigned long long key = ((unsigned long long)hsh(v) << 20) | (unsigned)best;
        if (p.kb == 1) atomicMin(Kc + cc, key);
        else {
          ulonglong2 cur = KB[cc];
          if (key < cur.x) atomicMin(reinterpret_cast<unsigned long long*>(KB + cc), key);
        }
      }
    }
  }
  if (acc == 0x1234567) out[0] = acc;
}

int main() {
  const size_t N = 64000000, C = 20000000;
  int2* rec; int4* LE; int* comp; unsigned long long* Kc; ulonglong2* KB; unsigned* grab; int* out;
  CK(cudaMalloc(&rec, N * 8)); CK(cudaMalloc(&LE, N * 128)); CK(cudaMalloc(&comp, N * 4));
  CK(cudaMalloc(&Kc, C * 8)); CK(cudaMalloc(&KB, C * 16)); CK(cudaMalloc(&grab, 4)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(LE, 0, N * 128)); CK(cudaMemset(comp, 0, N * 4)); CK(cudaMemset(Kc, 0xff, C * 8)); CK(cudaMemset(KB, 0xff, C * 16));
  // records: v = s (all rows live, row order)
  {
    int2* h = (int2*)malloc(N * 8);
    for (size_t i = 0; i < N; ++i) h[i] = make_int2((int)i, 0);
    CK(cudaMemcpy(rec, h, N * 8, cudaMemcpyHostToDevice)); free(h);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct V { const char* name; P p; } vs[] = {
    {"full: ell+compv+4 gathers (win 6.4M) + KB16 offer", {1, 1, 4, 2, 0, 6400000, 2000000}},
    {"full with Kc8 atomicMin", {1, 1, 4, 1, 0, 6400000, 2000000}},
    {"no offer", {1, 1, 4, 0, 0, 6400000, 2000000}},
    {"no offer, no ELL", {0, 1, 4, 0, 0, 6400000, 2000000}},
    {"gathers only", {0, 0, 4, 0, 0, 6400000, 2000000}},
    {"gathers only, evict_last", {0, 0, 4, 0, 1, 6400000, 2000000}},
    {"full, gathers evict_last", {1, 1, 4, 2, 1, 6400000, 2000000}},
    {"full, win 1.6M", {1, 1, 4, 2, 0, 1600000, 2000000}},
    {"full, win 0.4M", {1, 1, 4, 2, 0, 400000, 2000000}},
    {"full, cwin 0.6M (C3-like)", {1, 1, 4, 2, 0, 6400000, 600000}},
    {"ell+compv only", {1, 1, 0, 0, 0, 6400000, 2000000}},
    {"full, 2 gathers", {1, 1, 2, 2, 0, 6400000, 2000000}},
    {"full, 8 gathers", {1, 1, 8, 2, 0, 6400000, 2000000}},
  };
  int nb = 148 * 5;
  for (auto& v : vs) {
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      CK(cudaMemset(grab, 0, 4));
      cudaEventRecord(e0);
      k_round<<<nb, 256>>>(rec, LE, comp, Kc, KB, N, v.p, grab, out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("%-55s %7.3f ms  (%.3g rows/s)\n", v.name, best, N / best * 1e3);
  }
  return 0;
}
