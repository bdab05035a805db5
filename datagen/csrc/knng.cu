// knng.cu -- exact k-NN graph builder for low-dimensional point sets (d <= 5),
// uniform-grid cell search.  INPUT GENERATOR ONLY: not part of the clustering
// hot path, shares no code with paper_2009_04552_b200/ or oracle/.
//
// Output convention: rows exclude self; fp64 distance
// sqrt(sum_t (x_t - y_t)^2) from fp32 coordinates, summed in dimension order
// without fused multiply-add (bit-identical to datagen/knn_cpu.py); each row is
// ordered by (fp64 distance, index) and stored as fp32 dist / int32 nbr.
//
// Exactness: a query q in cell c collects every point of the 3^D block around c
// whose distance is <= h' = h (1 - 1e-6); the block contains the whole ball of
// radius h' (cell coordinates are computed in fp64).  If at least k such points
// exist, the k nearest are among them (any point left out is farther than h').
// Otherwise the query is redone with rings of radius R = 2, 3, ... cells.

#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdint>
#include <cstdio>

namespace {

constexpr int kCandCap = 2048;  // candidates staged per cell block
constexpr int kWarpBuf = 512;   // per-warp selection buffer
constexpr int kWarps = 8;
constexpr int kFbCap = 8192;    // fallback buffer (per query, global)

__device__ __forceinline__ double dist64(const float* __restrict__ a, const float* __restrict__ b, int D) {
  double acc = 0.0;
  for (int t = 0; t < D; ++t) {
    const double df = __dsub_rn((double)a[t], (double)b[t]);
    acc = __dadd_rn(acc, __dmul_rn(df, df));
  }
  return __dsqrt_rn(acc);
}

__device__ __forceinline__ bool pair_less(double da, int ia, double db, int ib) {
  return da < db || (da == db && ia < ib);
}

struct GridParams {
  int D;
  int bits;        // bits per coordinate in the linear cell key
  double lo[8];
  double inv_h;
  int64_t n;
};

__device__ __forceinline__ long long cell_coord(float x, double lo, double inv_h) {
  return (long long)floor(((double)x - lo) * inv_h);
}

__global__ void k_cell_keys(const float* __restrict__ X, GridParams gp, unsigned long long* __restrict__ keys,
                            int32_t* __restrict__ ids, int* __restrict__ overflow) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < gp.n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long key = 0;
    const long long lim = 1ll << gp.bits;
    for (int t = 0; t < gp.D; ++t) {
      long long c = cell_coord(X[i * gp.D + t], gp.lo[t], gp.inv_h);
      if (c < 1 || c >= lim - 1) atomicExch(overflow, 1);  // keep a 1-cell margin
      c = c < 0 ? 0 : (c >= lim ? lim - 1 : c);
      key = (key << gp.bits) | (unsigned long long)c;
    }
    keys[i] = key;
    ids[i] = (int32_t)i;
  }
}

__global__ void k_run_flags(const unsigned long long* __restrict__ keys, int64_t n, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_run_starts(const unsigned long long* __restrict__ keys, const int32_t* __restrict__ flag,
                             const int32_t* __restrict__ pos, int64_t n, unsigned long long* __restrict__ ukey,
                             int64_t* __restrict__ ustart) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) {
      ukey[pos[i]] = keys[i];
      ustart[pos[i]] = i;
    }
}

__device__ __forceinline__ int64_t find_cell(const unsigned long long* __restrict__ ukey, int64_t ncell,
                                             unsigned long long key) {
  int64_t lo = 0, hi = ncell;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ukey[mid] < key) lo = mid + 1; else hi = mid;
  }
  return (lo < ncell && ukey[lo] == key) ? lo : -1;
}

// decode / re-encode neighbour keys with per-dimension offsets in [-R, R]
__device__ __forceinline__ unsigned long long neighbour_key(unsigned long long key, int D, int bits, int o, int R) {
  const int W = 2 * R + 1;
  const unsigned long long mask = (1ull << bits) - 1;
  unsigned long long out = 0;
  for (int t = 0; t < D; ++t) {
    const int sh = (D - 1 - t) * bits;
    long long c = (long long)((key >> sh) & mask);
    int div = 1;
    for (int u = t + 1; u < D; ++u) div *= W;
    const int off = (o / div) % W - R;
    c += off;
    if (c < 0 || c > (long long)mask) return ~0ull;
    out |= (unsigned long long)c << sh;
  }
  return out;
}

// warp-cooperative bitonic sort of buf[0..n2) (n2 power of two >= 32) by (d, id)
__device__ void warp_bitonic(double* d, int* id, int n2) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = lane; t < n2 / 2; t += 32) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool asc = ((lo & size) == 0);
        const double dl = d[lo], dh = d[hi];
        const int il = id[lo], ih = id[hi];
        const bool swap = asc ? pair_less(dh, ih, dl, il) : pair_less(dl, il, dh, ih);
        if (swap) { d[lo] = dh; d[hi] = dl; id[lo] = ih; id[hi] = il; }
      }
      __syncwarp();
    }
  }
}

__device__ void block_bitonic(double* d, int* id, int n2) {
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < n2 / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool asc = ((lo & size) == 0);
        const double dl = d[lo], dh = d[hi];
        const int il = id[lo], ih = id[hi];
        const bool swap = asc ? pair_less(dh, ih, dl, il) : pair_less(dl, il, dh, ih);
        if (swap) { d[lo] = dh; d[hi] = dl; id[lo] = ih; id[hi] = il; }
      }
      __syncthreads();
    }
  }
}

// one block per cell (grid-stride): stage the 3^D block's points in smem, then
// each warp selects the k nearest for the queries of the cell
template <int D>
__global__ void __launch_bounds__(kWarps * 32) k_cells(const float* __restrict__ X, const int32_t* __restrict__ sid,
                                                       const unsigned long long* __restrict__ ukey,
                                                       const int64_t* __restrict__ ustart, int64_t ncell, int64_t n,
                                                       int bits, double hq, int k, int32_t* __restrict__ nbr,
                                                       float* __restrict__ dist, int32_t* __restrict__ fb,
                                                       unsigned int* __restrict__ nfb) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double (*wd)[kWarpBuf] = reinterpret_cast<double (*)[kWarpBuf]>(smem_raw);
  int (*wi)[kWarpBuf] = reinterpret_cast<int (*)[kWarpBuf]>(smem_raw + sizeof(double) * kWarps * kWarpBuf);
  float* cx = reinterpret_cast<float*>(smem_raw + (sizeof(double) + sizeof(int)) * kWarps * kWarpBuf);
  int* cid = reinterpret_cast<int*>(cx + kCandCap * D);
  __shared__ int64_t nb_start[256];
  __shared__ int nb_len[256];
  __shared__ int ncand, nnb;
  constexpr int NB = D == 1 ? 3 : D == 2 ? 9 : D == 3 ? 27 : D == 4 ? 81 : 243;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t c = blockIdx.x; c < ncell; c += gridDim.x) {
    const unsigned long long key = ukey[c];
    if (threadIdx.x == 0) nnb = 0;
    __syncthreads();
    for (int o = threadIdx.x; o < NB; o += blockDim.x) {
      const unsigned long long nk = neighbour_key(key, D, bits, o, 1);
      if (nk == ~0ull) continue;
      const int64_t j = find_cell(ukey, ncell, nk);
      if (j < 0) continue;
      const int s = atomicAdd(&nnb, 1);
      nb_start[s] = ustart[j];
      nb_len[s] = (int)((j + 1 < ncell ? ustart[j + 1] : n) - ustart[j]);
    }
    __syncthreads();
    // stage candidates (cooperative copy of every neighbour cell's points)
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int s = 0; s < nnb; ++s) tot += nb_len[s];
      ncand = tot;
    }
    __syncthreads();
    const int64_t qbeg = ustart[c], qend = (c + 1 < ncell ? ustart[c + 1] : n);
    if (ncand > kCandCap) {  // too dense: every query of this cell goes to the fallback
      for (int64_t q = qbeg + threadIdx.x; q < qend; q += blockDim.x) fb[atomicAdd(nfb, 1u)] = sid[q];
      __syncthreads();
      continue;
    }
    {
      int base = 0;
      for (int s = 0; s < nnb; ++s) {
        for (int t = threadIdx.x; t < nb_len[s]; t += blockDim.x) {
          const int32_t p = sid[nb_start[s] + t];
          cid[base + t] = p;
          for (int u = 0; u < D; ++u) cx[(base + t) * D + u] = X[(int64_t)p * D + u];
        }
        base += nb_len[s];
      }
    }
    __syncthreads();
    for (int64_t q = qbeg + warp; q < qend; q += kWarps) {
      const int32_t qi = sid[q];
      float qx[D];
      for (int u = 0; u < D; ++u) qx[u] = X[(int64_t)qi * D + u];
      int cnt = 0;
      bool over = false;
      for (int b0 = 0; b0 < ncand; b0 += 32) {
        const int t = b0 + lane;
        bool take = false;
        double dd = 0.0;
        int pid = -1;
        if (t < ncand) {
          pid = cid[t];
          if (pid != qi) {
            dd = dist64(qx, cx + t * D, D);
            take = dd <= hq;
          }
        }
        const unsigned m = __ballot_sync(0xffffffffu, take);
        const int pos = cnt + __popc(m & ((1u << lane) - 1u));
        if (take && pos < kWarpBuf) { wd[warp][pos] = dd; wi[warp][pos] = pid; }
        cnt += __popc(m);
      }
      over = cnt > kWarpBuf;
      if (cnt < k || over) {
        if (lane == 0) fb[atomicAdd(nfb, 1u)] = qi;
        __syncwarp();
        continue;
      }
      int n2 = 32;
      while (n2 < cnt) n2 <<= 1;
      for (int t = cnt + lane; t < n2; t += 32) { wd[warp][t] = 1e300; wi[warp][t] = 0x7fffffff; }
      __syncwarp();
      warp_bitonic(wd[warp], wi[warp], n2);
      for (int t = lane; t < k; t += 32) {
        nbr[(int64_t)qi * k + t] = wi[warp][t];
        dist[(int64_t)qi * k + t] = (float)wd[warp][t];
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

// fallback: one block per query, rings of radius R = 2, 4, 8, ... cells.  Pass 1
// histograms the distances <= R h' of the (2R+1)^D block into kHist linear
// buckets; the first bucket j where the cumulative count reaches k bounds the k
// nearest (bucket index is monotone in d); pass 2 collects buckets <= j, sorts
// them by (d, id) and writes the first k.
constexpr int kHist = 1024;
template <int D>
__global__ void __launch_bounds__(256) k_fallback(const float* __restrict__ X, const int32_t* __restrict__ sid,
                                                  const unsigned long long* __restrict__ ukey,
                                                  const int64_t* __restrict__ ustart, int64_t ncell, int64_t n, int bits,
                                                  double hq, double lo0, double lo1, double lo2, double lo3, double lo4,
                                                  double inv_h, int k, const int32_t* __restrict__ fb, unsigned nfb,
                                                  int32_t* __restrict__ nbr, float* __restrict__ dist,
                                                  int* __restrict__ fail, int max_ring, double diag) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* sd = reinterpret_cast<double*>(smem);
  int* si = reinterpret_cast<int*>(sd + kFbCap);
  __shared__ unsigned int hist[kHist];
  __shared__ int cnt, sel, total;
  const double lo[5] = {lo0, lo1, lo2, lo3, lo4};
  for (unsigned f = blockIdx.x; f < nfb; f += gridDim.x) {
    const int32_t qi = fb[f];
    float qx[D];
    for (int u = 0; u < D; ++u) qx[u] = X[(int64_t)qi * D + u];
    unsigned long long key = 0;
    for (int u = 0; u < D; ++u) key = (key << bits) | (unsigned long long)cell_coord(qx[u], lo[u], inv_h);
    for (int R = 2;; R *= 2) {
      long long W = 1;
      for (int u = 0; u < D; ++u) W *= (2 * R + 1);
      // beyond a few thousand cells (or the grid extent) scan every point instead
      const bool brute = R >= max_ring || W > 4096;
      const bool last = brute;
      for (int t = threadIdx.x; t < kHist; t += blockDim.x) hist[t] = 0;
      if (threadIdx.x == 0) { cnt = 0; total = 0; }
      __syncthreads();
      const double rq = brute ? diag : hq * R;
      const double scale = kHist / rq;
      for (int pass = 0; pass < 2; ++pass) {
        for (long long o = 0; o < (brute ? 1 : W); ++o) {  // cells sequentially, points in parallel
          int64_t b = 0, e = n;
          if (!brute) {
            const unsigned long long nk = neighbour_key(key, D, bits, (int)o, R);
            if (nk == ~0ull) continue;
            const int64_t j = find_cell(ukey, ncell, nk);
            if (j < 0) continue;
            b = ustart[j];
            e = (j + 1 < ncell ? ustart[j + 1] : n);
          }
          for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x) {
            const int32_t p = sid[t];
            if (p == qi) continue;
            const double dd = dist64(qx, X + (int64_t)p * D, D);
            if (!(dd <= rq)) continue;
            int bk = (int)(dd * scale);
            bk = bk >= kHist ? kHist - 1 : bk;
            if (pass == 0) {
              atomicAdd(&hist[bk], 1u);
            } else if (bk <= sel) {
              const int s = atomicAdd(&cnt, 1);
              if (s < kFbCap) { sd[s] = dd; si[s] = p; }
            }
          }
        }
        __syncthreads();
        if (pass == 0) {
          if (threadIdx.x == 0) {
            unsigned c = 0;
            int j = kHist - 1;
            for (int t = 0; t < kHist; ++t) {
              c += hist[t];
              if (c >= (unsigned)k) { j = t; break; }
            }
            unsigned tot = 0;
            for (int t = 0; t < kHist; ++t) tot += hist[t];
            sel = j;
            total = (int)tot;
          }
          __syncthreads();
          if (total < k && !last) break;  // grow the ring
        }
      }
      __syncthreads();
      if (total < k && !last) continue;
      const int c = cnt;
      if (c > kFbCap) { if (threadIdx.x == 0) atomicExch(fail, 1); break; }
      int n2 = 32;
      while (n2 < c) n2 <<= 1;
      for (int t = c + threadIdx.x; t < n2; t += blockDim.x) { sd[t] = 1e300; si[t] = -1; }
      __syncthreads();
      block_bitonic(sd, si, n2);
      for (int t = threadIdx.x; t < k; t += blockDim.x) {
        nbr[(int64_t)qi * k + t] = t < c ? si[t] : -1;
        dist[(int64_t)qi * k + t] = t < c ? (float)sd[t] : __int_as_float(0x7f800000);
      }
      if (c < k && threadIdx.x == 0) atomicExch(fail, 2);
      __syncthreads();
      break;
    }
    __syncthreads();
  }
}

// radius estimate: per sample query, histogram of distances on a log ladder
// bucket = floor(4 * log2(d / r_lo)) clamped to [0, 63]
__global__ void k_ladder(const float* __restrict__ X, int64_t n, int D, const int32_t* __restrict__ samples, int S,
                         float r_lo, unsigned int* __restrict__ hist) {
  __shared__ unsigned int sh[32][64];
  __shared__ float sq[32][8];
  for (int s0 = 0; s0 < S; s0 += 32) {
    const int ns = min(32, S - s0);
    for (int t = threadIdx.x; t < 32 * 64; t += blockDim.x) (&sh[0][0])[t] = 0;
    for (int t = threadIdx.x; t < ns * D; t += blockDim.x) sq[t / D][t % D] = X[(int64_t)samples[s0 + t / D] * D + t % D];
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      float p[8];
      for (int u = 0; u < D; ++u) p[u] = X[i * D + u];
      for (int s = 0; s < ns; ++s) {
        float d2 = 0.f;
        for (int u = 0; u < D; ++u) { const float df = p[u] - sq[s][u]; d2 += df * df; }
        int b = (int)floorf(2.0f * log2f(fmaxf(d2, 1e-30f) / (r_lo * r_lo)));
        b = b < 0 ? 0 : (b > 63 ? 63 : b);
        atomicAdd(&sh[s][b], 1u);
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ns * 64; t += blockDim.x)
      if ((&sh[0][0])[t]) atomicAdd(hist + (int64_t)(s0 + t / 64) * 64 + t % 64, (&sh[0][0])[t]);
    __syncthreads();
  }
}

}  // namespace

extern "C" {

// workspace bytes for knng_grid
size_t knng_grid_ws(int64_t n) {
  size_t tmp_sort = 0, tmp_scan = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  const size_t tmp = (tmp_sort > tmp_scan ? tmp_sort : tmp_scan) + 256;
  return 2 * n * 8 + 2 * n * 4 + n * 4 + n * 4 + n * 8 + n * 8 + n * 4 + tmp + 8 * 256;
}

// sample-based estimate of the k-th neighbour radius: returns per-sample upper
// bound of the bucket where the cumulative count first exceeds k (self counted)
int knng_ladder(const float* X, int64_t n, int D, const int32_t* samples, int S, float r_lo, unsigned int* hist,
                cudaStream_t st) {
  cudaMemsetAsync(hist, 0, (size_t)S * 64 * 4, st);
  k_ladder<<<148 * 4, 256, 0, st>>>(X, n, D, samples, S, r_lo, hist);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// build the exact kNN graph. returns 0 ok, 1 cuda error, 2 grid overflow (h too
// small for the bounding box), 3 fallback capacity exceeded, 4 bad args.
int knng_grid(const float* X, int64_t n, int D, int k, double h, const double* lo, double span_cells, double diag,
              int32_t* nbr, float* dist, void* ws, size_t ws_bytes, cudaStream_t st, int64_t* n_fallback) {
  if (D < 1 || D > 5 || k < 1 || k > n - 1 || !(h > 0)) return 4;
  if (ws_bytes < knng_grid_ws(n)) return 4;
  char* p = (char*)ws;
  auto take = [&](size_t b) { char* r = p; p += (b + 255) & ~size_t(255); return (void*)r; };
  unsigned long long* keys = (unsigned long long*)take(n * 8);
  unsigned long long* skeys = (unsigned long long*)take(n * 8);
  int32_t* ids = (int32_t*)take(n * 4);
  int32_t* sid = (int32_t*)take(n * 4);
  int32_t* flag = (int32_t*)take(n * 4);
  int32_t* pos = (int32_t*)take(n * 4);
  unsigned long long* ukey = (unsigned long long*)take(n * 8);
  int64_t* ustart = (int64_t*)take(n * 8);
  int32_t* fb = (int32_t*)take(n * 4);
  int* flags = (int*)take(256);
  size_t tmp_bytes = ws_bytes - (size_t)(p - (char*)ws);
  void* tmp = take(0);
  GridParams gp;
  gp.D = D;
  gp.bits = 63 / D;
  if (gp.bits > 21) gp.bits = 21;
  for (int t = 0; t < D; ++t) gp.lo[t] = lo[t];
  gp.inv_h = 1.0 / h;
  gp.n = n;
  cudaMemsetAsync(flags, 0, 256, st);
  const int G = 148 * 8;
  k_cell_keys<<<G, 256, 0, st>>>(X, gp, keys, ids, flags);
  size_t tb = tmp_bytes;
  if (cub::DeviceRadixSort::SortPairs(tmp, tb, keys, skeys, ids, sid, (int)n, 0, D * gp.bits, st)) return 1;
  k_run_flags<<<G, 256, 0, st>>>(skeys, n, flag);
  tb = tmp_bytes;
  if (cub::DeviceScan::ExclusiveSum(tmp, tb, flag, pos, (int)n, st)) return 1;
  k_run_starts<<<G, 256, 0, st>>>(skeys, flag, pos, n, ukey, ustart);
  int last[2];
  cudaMemcpyAsync(&last[0], pos + n - 1, 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&last[1], flag + n - 1, 4, cudaMemcpyDeviceToHost, st);
  int ovf = 0;
  cudaMemcpyAsync(&ovf, flags, 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return 1;
  if (ovf) return 2;
  const int64_t ncell = (int64_t)last[0] + last[1];
  const double hq = h * (1.0 - 1e-6);
  unsigned int* nfb = (unsigned int*)(flags + 4);
  const int gcells = (int)(ncell < 148 * 16 ? ncell : 148 * 16);
#define CELLS(DD)                                                                                          \
  {                                                                                                        \
    const int sm = (int)((sizeof(double) + sizeof(int)) * kWarps * kWarpBuf + (sizeof(float) * DD + 4) * kCandCap); \
    cudaFuncSetAttribute(k_cells<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);                    \
    k_cells<DD><<<gcells, kWarps * 32, sm, st>>>(X, sid, ukey, ustart, ncell, n, gp.bits, hq, k, nbr, dist, fb, nfb); \
  }
  switch (D) {
    case 1: CELLS(1) break;
    case 2: CELLS(2) break;
    case 3: CELLS(3) break;
    case 4: CELLS(4) break;
    case 5: CELLS(5) break;
  }
#undef CELLS
  if (cudaGetLastError() != cudaSuccess) return 1;
  unsigned int hfb = 0;
  cudaMemcpyAsync(&hfb, nfb, 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return 1;
  *n_fallback = hfb;
  if (hfb) {
    const size_t sm = (size_t)kFbCap * (8 + 4);
    int* fail = flags + 8;
    const double l[5] = {gp.lo[0], D > 1 ? gp.lo[1] : 0, D > 2 ? gp.lo[2] : 0, D > 3 ? gp.lo[3] : 0, D > 4 ? gp.lo[4] : 0};
    const int gf = (int)(hfb < 148 * 4 ? hfb : 148 * 4);
    // grid extent in cells (rings beyond it add nothing) and a distance bound
    const double ext = span_cells, dg = diag;
    int max_ring = 2;
    while (max_ring < ext) max_ring *= 2;
#define FB(DD)                                                                                                   \
  cudaFuncSetAttribute(k_fallback<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);                    \
  k_fallback<DD><<<gf, 256, sm, st>>>(X, sid, ukey, ustart, ncell, n, gp.bits, hq, l[0], l[1], l[2], l[3], l[4], \
                                      gp.inv_h, k, fb, hfb, nbr, dist, fail, max_ring, dg * 1.000001 + 1e-30);
    switch (D) {
      case 1: FB(1) break;
      case 2: FB(2) break;
      case 3: FB(3) break;
      case 4: FB(4) break;
      case 5: FB(5) break;
    }
#undef FB
    int hfail = 0;
    cudaMemcpyAsync(&hfail, fail, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return 1;
    if (hfail) return 3;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // extern "C"
