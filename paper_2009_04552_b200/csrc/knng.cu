// knng.cu -- exact k-NN graph builders (C-ABI in
// include/knng.h).  The stage that precedes clustering (Table 2,
// PAPER.md:21-36 times GOFMM's approximate builder); shares no code with the
// clustering kernels (kdb.cu) or the oracle.
//
// Output convention: rows exclude self; fp64 distance
// sqrt(sum_t (x_t - y_t)^2) from fp32 coordinates, summed in dimension order
// without fused multiply-add (bit-identical to datagen/knn_cpu.py); each row is
// ordered by (fp64 distance, index) and stored as fp32 dist / int32 nbr.
//
// Grid builder exactness: a query q in cell c collects every point of the 3^D
// block around c whose distance is <= h' = h (1 - 1e-6); the block contains the
// whole ball of radius h' (cell coordinates are computed in fp64).  If at least
// k such points exist, the k nearest are among them (any point left out is
// farther than h').  Otherwise the query is redone with rings of radius
// R = 2, 3, ... cells.

#include <cuda_runtime.h>

#include "knng.h"

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
                                                       unsigned int* __restrict__ nfb, int64_t qb, int64_t qe) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double (*wd)[kWarpBuf] = reinterpret_cast<double (*)[kWarpBuf]>(smem_raw);
  int (*wi)[kWarpBuf] = reinterpret_cast<int (*)[kWarpBuf]>(smem_raw + sizeof(double) * kWarps * kWarpBuf);
  float* cx = reinterpret_cast<float*>(smem_raw + (sizeof(double) + sizeof(int)) * kWarps * kWarpBuf);
  int* cid = reinterpret_cast<int*>(cx + kCandCap * D);
  __shared__ int64_t nb_start[256];
  __shared__ int nb_len[256];
  __shared__ int nb_pre[256];
  __shared__ int ncand, nnb;
  constexpr int NB = D == 1 ? 3 : D == 2 ? 9 : D == 3 ? 27 : D == 4 ? 81 : 243;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t c = blockIdx.x; c < ncell; c += gridDim.x) {
    const unsigned long long key = ukey[c];
    {
      // query rows [qb, qe) only: ids inside a cell are ascending (stable key
      // sort of 0..n-1), so a cell without such a query is skipped whole
      const int64_t b0 = ustart[c], e0 = (c + 1 < ncell ? ustart[c + 1] : n);
      if (sid[b0] >= qe || sid[e0 - 1] < qb) continue;  // block-uniform
    }
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
    // neighbour cells' points are staged in chunks of kCandCap (5-D blocks of
    // 3^5 cells often hold more); each warp accumulates its query's points
    // within h' over all chunks
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int s2 = 0; s2 < nnb; ++s2) { nb_pre[s2] = tot; tot += nb_len[s2]; }
      ncand = tot;
    }
    __syncthreads();
    const int64_t qbeg = ustart[c], qend = (c + 1 < ncell ? ustart[c + 1] : n);
    const bool one_chunk = ncand <= kCandCap;
    auto stage = [&](int cbase) {
      const int cend = min(cbase + kCandCap, ncand);
      for (int s2 = 0; s2 < nnb; ++s2) {
        const int lo = max(nb_pre[s2], cbase), hi = min(nb_pre[s2] + nb_len[s2], cend);
        for (int f = lo + (int)threadIdx.x; f < hi; f += blockDim.x) {
          const int32_t p = sid[nb_start[s2] + (f - nb_pre[s2])];
          cid[f - cbase] = p;
          for (int u = 0; u < D; ++u) cx[(f - cbase) * D + u] = X[(int64_t)p * D + u];
        }
      }
    };
    if (one_chunk) stage(0);
    __syncthreads();
    for (int64_t q0 = qbeg; q0 < qend; q0 += kWarps) {
      const int64_t q = q0 + warp;
      const int32_t q_id = q < qend ? sid[q] : -1;
      const bool active = q < qend && q_id >= qb && q_id < qe;
      const int32_t qi = active ? q_id : -1;
      float qx[D];
      for (int u = 0; u < D; ++u) qx[u] = active ? X[(int64_t)qi * D + u] : 0.f;
      int cnt = 0;
      for (int cbase = 0; cbase < ncand; cbase += kCandCap) {
        if (!one_chunk) {
          __syncthreads();
          stage(cbase);
          __syncthreads();
        }
        const int cn = min(kCandCap, ncand - cbase);
        if (!active) continue;
        for (int b0 = 0; b0 < cn; b0 += 32) {
          const int t = b0 + lane;
          bool take = false;
          double dd = 0.0;
          int pid = -1;
          if (t < cn) {
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
      }
      if (!active) continue;
      if (cnt < k || cnt > kWarpBuf) {
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
        nbr[((int64_t)qi - qb) * k + t] = wi[warp][t];
        dist[((int64_t)qi - qb) * k + t] = (float)wd[warp][t];
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
                                                  int* __restrict__ fail, int max_ring, double diag, int64_t qb) {
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
        nbr[((int64_t)qi - qb) * k + t] = t < c ? si[t] : -1;
        dist[((int64_t)qi - qb) * k + t] = t < c ? (float)sd[t] : __int_as_float(0x7f800000);
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

// ============================================================================
// Any-d exact kNN by brute force (C2: d = 50, C3: d = 10) -- input
// construction, not the hot path.  Pass 1 never materialises the N^2
// distances: each thread owns one query, streams every candidate through a
// shared-memory tile (rotated to start at the query's own id block, so the
// threshold drops early on cluster-major ids), computes the fp32
// difference-form squared distance and keeps the Kp smallest in a max-heap in
// global scratch.  Pass 2 recomputes the Kp candidates exactly (fp64, dimension
// order, no fusion -- the datagen/knn_cpu.py definition), sorts them by
// (distance, index) and keeps k.  Certificate: the fp32 sum of d squared
// differences is within a relative delta = (d + 3) 2^-24 of the real value, so
// if heap_max (1 - delta) > A (1 + delta), A = the largest fp32 value among the
// exact top-k, no point outside the heap can belong to the top-k.  Rows that
// fail it are flagged and recomputed exactly over all points.
constexpr int kBrT = 256;   // threads (= queries) per block
constexpr int kBrTile = 128;

__device__ __forceinline__ void heap_sift(float* hs, int32_t* hi, int n, int p) {
  while (true) {
    const int l = 2 * p + 1, r = l + 1;
    int m = p;
    if (l < n && hs[l] > hs[m]) m = l;
    if (r < n && hs[r] > hs[m]) m = r;
    if (m == p) return;
    const float ts = hs[p]; hs[p] = hs[m]; hs[m] = ts;
    const int32_t ti = hi[p]; hi[p] = hi[m]; hi[m] = ti;
    p = m;
  }
}

template <int DC>  // DC > 0: compile-time dimension; 0: runtime d (<= 64)
__global__ void __launch_bounds__(kBrT) k_brute_cand(const float* __restrict__ X, int64_t n, int d_rt, int Kp,
                                                       float* __restrict__ hs_all, int32_t* __restrict__ hi_all,
                                                       int32_t* __restrict__ hcount) {
  constexpr int DM = DC > 0 ? DC : 64;
  const int D = DC > 0 ? DC : d_rt;
  __shared__ __align__(16) float tile[DM * kBrTile];  // [dim][candidate]
  const int64_t qi = (int64_t)blockIdx.x * kBrT + threadIdx.x;
  const bool active = qi < n;
  float q[DM];
#pragma unroll
  for (int t = 0; t < DM; ++t) q[t] = (active && t < D) ? X[qi * D + t] : 0.f;
  float* hs = hs_all + (active ? qi : 0) * Kp;
  int32_t* hi = hi_all + (active ? qi : 0) * Kp;
  int h = 0;
  float thr = __int_as_float(0x7f800000);
  const int64_t ntiles = (n + kBrTile - 1) / kBrTile;
  const int64_t t_start = ((int64_t)blockIdx.x * kBrT) / kBrTile;
  for (int64_t tt = 0; tt < ntiles; ++tt) {
    const int64_t tile_id = (t_start + tt) % ntiles;
    const int64_t c0 = tile_id * kBrTile;
    const int nc = (int)min((int64_t)kBrTile, n - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < kBrTile * D; e += kBrT) {
      const int c = e / D, t = e - c * D;
      tile[t * kBrTile + c] = c < nc ? __ldg(X + (c0 + c) * D + t) : 0.f;
    }
    __syncthreads();
    if (!active) continue;
    for (int c = 0; c < nc; c += 4) {
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int t = 0; t < DM; ++t) {
        if (DC == 0 && t >= D) break;
        const float4 x = *reinterpret_cast<const float4*>(tile + t * kBrTile + c);
        const float a0 = q[t] - x.x, a1 = q[t] - x.y, a2 = q[t] - x.z, a3 = q[t] - x.w;
        s0 = fmaf(a0, a0, s0);
        s1 = fmaf(a1, a1, s1);
        s2 = fmaf(a2, a2, s2);
        s3 = fmaf(a3, a3, s3);
      }
      const float sv[4] = {s0, s1, s2, s3};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int64_t j = c0 + c + r;
        if (c + r >= nc || j == qi || !(sv[r] < thr)) continue;
        if (h < Kp) {
          hs[h] = sv[r];
          hi[h] = (int32_t)j;
          if (++h == Kp) {
            for (int p2 = Kp / 2 - 1; p2 >= 0; --p2) heap_sift(hs, hi, Kp, p2);
            thr = hs[0];
          }
        } else {
          hs[0] = sv[r];
          hi[0] = (int32_t)j;
          heap_sift(hs, hi, Kp, 0);
          thr = hs[0];
        }
      }
    }
  }
  if (active) hcount[qi] = h;
}

__device__ __forceinline__ double exact_d64(const float* __restrict__ a, const float* __restrict__ b, int D) {
  double acc = 0.0;
  for (int t = 0; t < D; ++t) {
    const double df = __dsub_rn((double)a[t], (double)b[t]);
    acc = __dadd_rn(acc, __dmul_rn(df, df));
  }
  return sqrt(acc);
}

// one warp per query: exact fp64 distances of the heap, bitonic sort by
// (distance, index) in shared memory, top k out, certificate check
constexpr int kRrWarps = 8;
constexpr int kRrBuf = 256;  // Kp <= 256
__global__ void __launch_bounds__(kRrWarps * 32) k_brute_rerank(const float* __restrict__ X, int64_t n, int D, int k,
                                                                 int Kp, const float* __restrict__ hs_all,
                                                                 const int32_t* __restrict__ hi_all,
                                                                 const int32_t* __restrict__ hcount,
                                                                 int32_t* __restrict__ nbr, float* __restrict__ dist,
                                                                 int32_t* __restrict__ fail_rows,
                                                                 unsigned int* __restrict__ n_fail) {
  __shared__ double sd[kRrWarps][kRrBuf];
  __shared__ int si[kRrWarps][kRrBuf];
  __shared__ float ss[kRrWarps][kRrBuf];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double delta = (D + 3) * 5.9604644775390625e-8;  // (d + 3) 2^-24
  for (int64_t qi = (int64_t)blockIdx.x * kRrWarps + w; qi < n; qi += (int64_t)gridDim.x * kRrWarps) {
    const int h = hcount[qi];
    const float* hs = hs_all + qi * Kp;
    const int32_t* hi = hi_all + qi * Kp;
    float hmax = 0.f;
    for (int e = lane; e < kRrBuf; e += 32) {
      if (e < h) {
        const int32_t j = hi[e];
        sd[w][e] = exact_d64(X + qi * D, X + (int64_t)j * D, D);
        si[w][e] = j;
        ss[w][e] = hs[e];
        hmax = fmaxf(hmax, hs[e]);
      } else {
        sd[w][e] = __longlong_as_double(0x7ff0000000000000ll);
        si[w][e] = 0x7fffffff;
        ss[w][e] = 0.f;
      }
    }
    for (int o = 16; o > 0; o >>= 1) hmax = fmaxf(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
    __syncwarp();
    // bitonic sort of kRrBuf entries by (distance, index)
    for (int size = 2; size <= kRrBuf; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int e = lane; e < kRrBuf / 2; e += 32) {
          const int lo = 2 * e - (e & (stride - 1)), hi2 = lo + stride;
          const bool up = (lo & size) == 0;
          const double dl = sd[w][lo], dh = sd[w][hi2];
          const int il = si[w][lo], ih = si[w][hi2];
          const bool gt = dl > dh || (dl == dh && il > ih);
          if (gt == up) {
            sd[w][lo] = dh; sd[w][hi2] = dl;
            si[w][lo] = ih; si[w][hi2] = il;
            const float t = ss[w][lo]; ss[w][lo] = ss[w][hi2]; ss[w][hi2] = t;
          }
        }
        __syncwarp();
      }
    }
    float amax = 0.f;
    for (int e = lane; e < k; e += 32) {
      nbr[qi * k + e] = si[w][e];
      dist[qi * k + e] = (float)sd[w][e];
      amax = fmaxf(amax, ss[w][e]);
    }
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    // a heap that never filled saw every other point: exact without a certificate
    const bool ok = h < Kp || (double)hmax * (1.0 - delta) > (double)amax * (1.0 + delta);
    if (!ok && lane == 0) fail_rows[atomicAdd(n_fail, 1u)] = (int32_t)qi;
    __syncwarp();
  }
}

// exact fp64 distances from query row q to every point (fallback rows)
__global__ void k_exact_row(const float* __restrict__ X, int64_t n, int D, int64_t q, double* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    out[j] = j == q ? __longlong_as_double(0x7ff0000000000000ll) : exact_d64(X + q * D, X + j * D, D);
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
int knng_grid_rows(const float* X, int64_t n, int D, int k, double h, const double* lo, double span_cells,
                   double diag, int64_t q_begin, int64_t q_count, int32_t* nbr, float* dist, void* ws,
                   size_t ws_bytes, cudaStream_t st, int64_t* n_fallback) {
  if (D < 1 || D > 5 || k < 1 || k > n - 1 || !(h > 0)) return 4;
  if (q_begin < 0 || q_count < 0 || q_begin + q_count > n) return 4;
  if (q_count == 0) { *n_fallback = 0; return 0; }
  const int64_t qb = q_begin, qe = q_begin + q_count;
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
    k_cells<DD><<<gcells, kWarps * 32, sm, st>>>(X, sid, ukey, ustart, ncell, n, gp.bits, hq, k, nbr, dist, fb, nfb, \
                                                 qb, qe);                                                  \
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
                                      gp.inv_h, k, fb, hfb, nbr, dist, fail, max_ring, dg * 1.000001 + 1e-30, qb);
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

int knng_grid(const float* X, int64_t n, int D, int k, double h, const double* lo, double span_cells, double diag,
              int32_t* nbr, float* dist, void* ws, size_t ws_bytes, cudaStream_t st, int64_t* n_fallback) {
  return knng_grid_rows(X, n, D, k, h, lo, span_cells, diag, 0, n, nbr, dist, ws, ws_bytes, st, n_fallback);
}

// brute-force candidates + exact re-rank; rows failing the certificate are
// written to fail_rows (count in *n_fail) for knng_exact_row.  scratch: n*Kp
// floats + n*Kp ints + n ints.  Returns 0 ok, 1 cuda error, 4 bad args.
int knng_brute(const float* X, int64_t n, int D, int k, int Kp, float* hs, int32_t* hi, int32_t* hcount,
               int32_t* nbr, float* dist, int32_t* fail_rows, unsigned int* n_fail, cudaStream_t st) {
  if (D < 1 || D > 64 || k < 1 || k > n - 1 || Kp < k || Kp > kRrBuf) return 4;
  const int g = (int)((n + kBrT - 1) / kBrT);
  if (D == 10)
    k_brute_cand<10><<<g, kBrT, 0, st>>>(X, n, D, Kp, hs, hi, hcount);
  else if (D == 50)
    k_brute_cand<50><<<g, kBrT, 0, st>>>(X, n, D, Kp, hs, hi, hcount);
  else
    k_brute_cand<0><<<g, kBrT, 0, st>>>(X, n, D, Kp, hs, hi, hcount);
  if (cudaGetLastError() != cudaSuccess) return 1;
  cudaMemsetAsync(n_fail, 0, 4, st);
  k_brute_rerank<<<148 * 16, kRrWarps * 32, 0, st>>>(X, n, D, k, Kp, hs, hi, hcount, nbr, dist, fail_rows, n_fail);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int knng_exact_row(const float* X, int64_t n, int D, int64_t q, double* out, cudaStream_t st) {
  k_exact_row<<<148 * 4, 256, 0, st>>>(X, n, D, q, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // extern "C"
