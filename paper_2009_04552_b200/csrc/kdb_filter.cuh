// kdb_filter.cuh -- Filter-Boruvka kernels: light threshold, filter fast path, heavy phase, inexact-MST kernels
// Part of kdb.cu's single translation unit: included inside its anonymous
// namespace, after kdb.cu's helpers; not a standalone header.
#pragma once

// ============================================================================
// Filter-Boruvka: light phase, filter, heavy phase
// ============================================================================
// The rounds above run first on the LIGHT candidate graph G_L = entries with
// w <= tau (tau < eps, sampled so that G_L's components are large).  Every
// light key is smaller than every heavy key (mono(w) is the major field of
// O1), so by the cut and cycle properties
//     MSF(G) = MSF(G_L)  U  MSF(G / comp_L restricted to heavy entries whose
//                              endpoints lie in different light components).
// k_filter streams the heavy entries once and keeps only those that cross
// light components ("survivors"); the heavy phase runs edge-centric Boruvka on
// the survivors in the contracted (component) space, where every survivor is
// offered to both endpoint components -- undirected by construction, so it is
// exact for ANY valid graph (no certificate, no in-edge lists).

// tau sampling: column `col` of every stride-th local row
__global__ void k_sample_col(const float* __restrict__ dist, int64_t n_rows, int32_t ld, int32_t col, int64_t stride,
                             int64_t n_out, float* __restrict__ out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_out; s += (int64_t)gridDim.x * blockDim.x)
    out[s] = __ldg(dist + (s * stride) * ld + col);
}

struct HEdge {     // a survivor: a heavy candidate entry that crosses light components
  uint64_t key;    // (mono(w) << 32) | a
  int32_t x, y;    // light-component ids of the row vertex and of the target J
  uint32_t b;      // max endpoint
  uint32_t pad;
};
static_assert(sizeof(HEdge) == 24, "HEdge layout");

// ---------------------------------------------------------------------------
// Filter fast path (exact).  Most heavy entries join two vertices of the same
// light component, and ids are block-local (points of a cluster have nearby
// ids), so the per-entry component gather is replaced by two shared-memory
// probes:  id block J >> dom_shift has a dominant component dom[blk]; the
// exceptions X = {x core : comp[x] != dom[x >> dom_shift]} go into a Bloom
// filter (no false negatives).  If dom[J >> shift] == comp[v] and J is not
// (possibly) in X, then comp[J] == comp[v] and the entry is intra -- skipped
// without touching comp[].  Everything else takes the exact gather.
constexpr int kDomMax = 16384;         // dom table entries (64 KB of shared memory)
constexpr int kBloomBits = 1 << 20;    // 128 KB of shared memory
#ifndef KDB_FILTER_THREADS
#define KDB_FILTER_THREADS 1024
#endif
#ifndef KDB_FILTER_UNROLL
#define KDB_FILTER_UNROLL 4
#endif
#ifndef KDB_FILTER_PREFETCH
#define KDB_FILTER_PREFETCH 1
#endif
constexpr int kFilterThreads = KDB_FILTER_THREADS;  // threads per block
constexpr int kFilterUnroll = KDB_FILTER_UNROLL;    // 16-B id chunks in flight per thread
// Each WARP sweeps its own tiles of 32 x unroll rows (a tile of ld-entry rows
// is exactly ld / VEC sweep steps), staged in its own slice of shared memory:
// no block barrier after the Bloom copy, warps never wait for each other.
constexpr int kFilterRows = 32 * kFilterUnroll;  // rows per warp tile
constexpr int kFilterWarps = kFilterThreads / 32;
constexpr size_t kFilterSmem = kBloomBits / 8 + (size_t)kFilterWarps * kFilterRows * 16;  // Bloom words, then each warp's FRow tile

// Blocked Bloom filter: key x selects ONE 32-bit word and sets 2-4 bits in it:
// a single shared-memory probe per test.  One multiplicative hash h = x * phi
// serves both: the word from its top 15 bits, the bits from two rotations
// by bits [0,5) and [5,10) (the low bits of h are a bijection of the low bits
// of x, independent of the word choice).  At C4 (18,301 keys) 9.5M of 6.4G
// entries take the slow path (8.4M with three independent bits, which cost
// two more instructions per entry: filter 7.18 -> 6.92 ms).
__device__ __forceinline__ uint32_t bloom_hash(uint32_t x) { return x * 0x9E3779B1u; }
__device__ __forceinline__ uint32_t bloom_word_h(uint32_t h) { return h >> 17; }
// The word's mask: two fixed 2-bit patterns rotated by bits [0,5) and [5,10)
// of h (a rotate is one funnel shift): 2-4 bits set, 4 instructions.  One
// word per key makes the false-positive rate about (keys per word) / (distinct
// masks): a single rotation of one 3-bit pattern (32 masks) measured 103.6M
// slow entries at C4 against 9.5M with these 1,024 masks, and a 12.6 ms filter.
__device__ __forceinline__ uint32_t bloom_mask_h(uint32_t h) {
  constexpr uint32_t P1 = 1u | (1u << 11), P2 = 1u | (1u << 19);
  return __funnelshift_l(P1, P1, h) | __funnelshift_l(P2, P2, h >> 5);
}
__device__ __forceinline__ uint32_t bloom_word(uint32_t x) { return bloom_word_h(bloom_hash(x)); }
__device__ __forceinline__ uint32_t bloom_mask(uint32_t x) { return bloom_mask_h(bloom_hash(x)); }

// dom[blk]: majority component among 32 sampled vertices of the id block (-1 if none is core)
__global__ void k_dom(const int32_t* __restrict__ comp, int64_t N, int shift, int64_t nblk,
                      int32_t* __restrict__ dom) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t blk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; blk < nblk; blk += nw) {
    const int64_t lo = blk << shift, len = min((int64_t)1 << shift, N - lo);
    const int64_t x = lo + (len * lane) / 32;
    const int32_t c = x < N ? comp[x] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    int cnt = c >= 0 ? __popc(grp) : 0;
    int best = cnt, bc = c;
    for (int o = 16; o > 0; o >>= 1) {
      const int oc = __shfl_xor_sync(0xffffffffu, best, o);
      const int ob = __shfl_xor_sync(0xffffffffu, bc, o);
      if (oc > best || (oc == best && ob > bc)) { best = oc; bc = ob; }
    }
    if (lane == 0) dom[blk] = best > 0 ? bc : -1;
  }
}

__global__ void k_bloom_build(const int32_t* __restrict__ comp, int64_t N, int shift, const int32_t* __restrict__ dom,
                              uint32_t* __restrict__ bloom, uint32_t* __restrict__ n_exc) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < N; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = base + threadIdx.x;
    bool exc = false;
    if (x < N) {
      const int32_t c = comp[x];
      exc = c >= 0 && c != dom[x >> shift];
      if (exc) atomicOr(bloom + bloom_word((uint32_t)x), bloom_mask((uint32_t)x));
    }
    block_count(n_exc, exc);
  }
}

// per-component id range [lo, hi) made of a contiguous run of id blocks whose
// dominant component it is (else empty): rlo/rhi/rcnt are C-sized scratch
__global__ void k_rng_acc(const int32_t* __restrict__ dom, int64_t nblk, int32_t* __restrict__ rlo,
                          int32_t* __restrict__ rhi, int32_t* __restrict__ rcnt) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblk; b += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = dom[b];
    if (g < 0) continue;
    atomicMin(rlo + g, (int32_t)b);
    atomicMax(rhi + g, (int32_t)b);
    atomicAdd(rcnt + g, 1);
  }
}
__global__ void k_rng_fin(int64_t C, int64_t N, int shift, const int32_t* __restrict__ rlo,
                          const int32_t* __restrict__ rhi, const int32_t* __restrict__ rcnt, int2* __restrict__ rng) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C; c += (int64_t)gridDim.x * blockDim.x) {
    const int32_t n = rcnt[c], lo = rlo[c], hi = rhi[c];
    if (n > 0 && n == hi - lo + 1)
      rng[c] = make_int2((int32_t)((int64_t)lo << shift), (int32_t)min(((int64_t)hi + 1) << shift, N));
    else
      rng[c] = make_int2(1, 0);
  }
}

// q / d by one multiply-high (d > 1: M = ceil(2^64 / d); exact for q < 2^64 / d)
struct FastDiv {
  uint64_t M;
  uint64_t d;
  uint32_t m32;  // ceil(2^32 / d): n / d == umulhi(n, m32) for n < 2^32 / d
  uint32_t small;  // 1 < d < 2048: the 32-bit path is exact for the tile's indices
};
__device__ __forceinline__ uint64_t fdiv(uint64_t q, const FastDiv& f) { return f.d == 1 ? q : __umul64hi(q, f.M); }

// The filter: every rank streams its rows once, each warp in its own tiles of
// kFilterRows rows.  Per tile, the warp's lanes stage the rows' data in the
// warp's slice of shared memory (comp[v] and an id range of comp[v]: the
// component's whole range when its dominated blocks form one run, else the run
// of blocks dominated by comp[v] around v's own block, brun); then
// the tile's R*k ids are swept in flat order, VEC per lane and chunk.  Fast path: J inside the id range of comp[v] and
// not in the Bloom filter of the exceptions => comp[J] == comp[v]: the entry
// is intra (or light, or beyond eps, or J == v -- none a candidate leaving
// edge), decided from the id alone.  Otherwise the chunk's weights are loaded
// and a heavy (tau < w <= eps) candidate survives iff comp[J] != comp[v].
struct FRow {
  int32_t cr;     // comp[v] (< 0: non-core row)
  uint32_t lo;    // id range of comp[v]: [lo, lo + span)
  uint32_t span;
  uint32_t pad;
};

// COLS (edge_cols < row stride ld): only columns < k are candidates; the sweep
// enumerates just the ceil(k / VEC) chunks at the head of each row (fd then
// divides by that count), so columns >= k cost neither loads nor issue slots.
template <int VEC, bool FAST, bool COLS, bool SMALL = false>
__global__ void __launch_bounds__(kFilterThreads) k_filter(
    const int32_t* __restrict__ nbr, const float* __restrict__ dist, int64_t n_rows, int32_t ld, int32_t k, float tau, float eps,
    int64_t row_begin, int64_t N, const int32_t* __restrict__ comp, const int2* __restrict__ rng, const uint32_t* __restrict__ bloom, FastDiv fd,
    HEdge* __restrict__ out, uint32_t cap, uint32_t* __restrict__ n_out, unsigned long long* __restrict__ n_slow,
    const int32_t* __restrict__ dom, const int2* __restrict__ brun, int shift) {
  extern __shared__ uint32_t s_bloom[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  FRow* s_row = reinterpret_cast<FRow*>(s_bloom + kBloomBits / 32) + wid * kFilterRows;
  constexpr int R = kFilterRows;
  const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(s_bloom);
  if (FAST) {
    for (int t = threadIdx.x; t < kBloomBits / 32; t += blockDim.x) s_bloom[t] = bloom[t];
  }
  const uint32_t Nu = (uint32_t)N;
  const int64_t n_tiles = (n_rows + R - 1) / R;
  uint32_t slow = 0;
  __syncthreads();  // the Bloom copy is complete
  for (int64_t tile = (int64_t)blockIdx.x * kFilterWarps + wid; tile < n_tiles; tile += (int64_t)gridDim.x * kFilterWarps) {
    const int64_t r0 = tile * R;
    const int nr = (int)((n_rows - r0) < R ? (n_rows - r0) : R);
    __syncwarp();  // the warp's previous tile readers are done with its s_row slice
    for (int ti = lane; ti < nr; ti += 32) {
      const int64_t i = r0 + ti;
      FRow fr;
      fr.cr = __ldg(comp + row_begin + i);
      fr.lo = 0;
      fr.span = 0;
      if (FAST && fr.cr >= 0) {
        int2 rg = __ldg(rng + fr.cr);
        if (!(rg.y > rg.x)) {  // no single range: the run of blocks dominated by comp[v] around v
          const int64_t b = (row_begin + i) >> shift;
          if (__ldg(dom + b) == fr.cr) rg = __ldg(brun + b);
        }
        if (rg.y > rg.x) { fr.lo = (uint32_t)rg.x; fr.span = (uint32_t)(rg.y - rg.x); }
      }
      s_row[ti] = fr;
    }
    __syncwarp();
    const int32_t* __restrict__ nt = nbr + r0 * ld;  // this tile's ids (contiguous)
    const float* __restrict__ dt = dist + r0 * ld;
    const uint32_t cpr = (uint32_t)((k + VEC - 1) / VEC);  // COLS: chunks per row
    const uint32_t n_chunks = COLS ? (uint32_t)nr * cpr : (uint32_t)(((int64_t)nr * ld) / VEC);
    // kFilterUnroll chunks per thread and step: their id loads are issued
    // together (the sweep is bound by load latency x loads in flight)
    for (uint32_t base = 0; base < n_chunks; base += 32 * kFilterUnroll) {
      int32_t J[kFilterUnroll][VEC];
#pragma unroll
      for (int t = 0; t < kFilterUnroll; ++t) {
        // past the end (ragged last step only): reload the last chunk instead
        // of predicating the load -- the consumer skips u >= n_chunks anyway
        const uint32_t u = min(base + t * 32 + lane, n_chunks - 1);
        uint32_t off = u;  // chunk offset from the tile start
        if (COLS) {
          const uint32_t lr = SMALL ? __umulhi(u, fd.m32) : (uint32_t)fdiv(u, fd);
          off = lr * (uint32_t)(ld / VEC) + (u - lr * cpr);
        }
#if KDB_FILTER_PREFETCH
        {  // the next step's chunk into L2 (its load then waits on L2, not HBM)
          const uint32_t un = base + (t + KDB_FILTER_PREFETCH * kFilterUnroll) * 32 + lane;
          // chunk un starts at element un * VEC (byte-correct for VEC == 1 too)
          if (!COLS && un < n_chunks) asm volatile("prefetch.global.L2 [%0];" ::"l"(nt + (size_t)un * VEC));
        }
#endif
        if (VEC == 4) {
          const int4 j4 = __ldcs(reinterpret_cast<const int4*>(nt) + off);
          J[t][0] = j4.x; J[t][1] = j4.y; J[t][2] = j4.z; J[t][3] = j4.w;
        } else {
          J[t][0] = __ldcs(nt + off);
        }
      }
#pragma unroll
      for (int t = 0; t < kFilterUnroll; ++t) {
        const uint32_t u = base + t * 32 + lane;
        uint32_t survm = 0, lr = 0, col = 0, off = u;
        int32_t cj[VEC], cr = -1;
        float w[VEC];
        if (u < n_chunks) {
          if (COLS) {
            lr = SMALL ? __umulhi(u, fd.m32) : (uint32_t)fdiv(u, fd);  // row within the tile
            col = (u - lr * cpr) * VEC;
            off = lr * (uint32_t)(ld / VEC) + (u - lr * cpr);
          } else {
            const uint32_t n = u * VEC;
            lr = SMALL ? __umulhi(n, fd.m32) : (uint32_t)fdiv(n, fd);  // row within the tile
            col = n - lr * (uint32_t)ld;
          }
          const FRow fr = s_row[lr];
          cr = fr.cr;
          // Fast test first: J in the id range of comp[v] and not a possible
          // exception => comp[J] == comp[v].  That also settles light entries,
          // entries beyond eps and J == v (none is a candidate leaving edge), so
          // the full classification below only runs for the rare rest.
          uint32_t slowm = 0;
#pragma unroll
          for (int j = 0; j < VEC; ++j) {
            uint32_t fast = 0;
            if (FAST) {
              const uint32_t Jj = (uint32_t)J[t][j];
              const uint32_t hh = bloom_hash(Jj);
              uint32_t word;
              asm("ld.shared.u32 %0, [%1];" : "=r"(word) : "r"(s_base + bloom_word_h(hh) * 4u));
              const uint32_t bm = bloom_mask_h(hh);
              fast = (uint32_t)((Jj - fr.lo) < fr.span) & (uint32_t)((word & bm) != bm);
            }
            slowm |= ((fast & 1u) ^ 1u) << j;
          }
          if (COLS) slowm &= (1u << min((uint32_t)VEC, (uint32_t)k - col)) - 1u;
          if (fr.cr < 0) slowm = 0;  // non-core row: no candidate entries
          if (slowm) {
            const uint32_t v = (uint32_t)(row_begin + r0 + lr);
            if (VEC == 4) {
              const float4 w4 = __ldg(reinterpret_cast<const float4*>(dt) + off);
              w[0] = w4.x; w[1] = w4.y; w[2] = w4.z; w[3] = w4.w;
            } else {
              w[0] = __ldg(dt + off);
            }
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
              cj[j] = -1;
              const uint32_t Jj = (uint32_t)J[t][j];
              const bool heavy = w[j] > tau && w[j] <= eps;  // not light, and a candidate weight
              if (((slowm >> j) & 1u) && heavy && Jj < Nu && Jj != v) {
                ++slow;
                cj[j] = gat(comp + Jj);
                if (cj[j] >= 0 && cj[j] != cr) survm |= 1u << j;
              }
            }
          }
        }
        if (__any_sync(0xffffffffu, survm != 0)) {  // rare: warp-aggregated append
          const int cnt = __popc(survm);
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int x = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += x;
          }
          const int tot = __shfl_sync(0xffffffffu, incl, 31);
          uint32_t base_slot = 0;
          if (lane == 31) {
            base_slot = atomicAdd(n_out, (uint32_t)tot);
            // sticky overflow flag in n_out[1]: the 32-bit count itself could wrap
            if ((uint64_t)base_slot + (uint64_t)tot > (uint64_t)cap) atomicOr(n_out + 1, 1u);
          }
          base_slot = __shfl_sync(0xffffffffu, base_slot, 31);
          uint32_t slot = base_slot + (uint32_t)(incl - cnt);
#pragma unroll
          for (int j = 0; j < VEC; ++j) {
            if (!((survm >> j) & 1u)) continue;
            if (slot < cap) {
              const int64_t v = row_begin + r0 + lr;
              HEdge hh;
              hh.key = pack_key(mono_bits(w[j]), (uint32_t)min(v, (int64_t)J[t][j]));
              hh.b = (uint32_t)max(v, (int64_t)J[t][j]);
              hh.x = cr;
              hh.y = cj[j];
              hh.pad = 0;
              out[slot] = hh;
            }
            ++slot;
          }
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) slow += __shfl_xor_sync(0xffffffffu, slow, o);
  if ((threadIdx.x & 31) == 0 && slow) atomicAdd(n_slow, (unsigned long long)slow);
}

// ---- inexact MST (Alg. 2 + 4) -------
// Group of id x under the contiguous split lo_p = floor(p N / P).
__device__ __forceinline__ int part_of(int64_t x, int64_t N, int P) {
  int64_t p = (x * P) / N;
  if (((p + 1) * N) / P <= x) ++p;
  else if ((p * N) / P > x) --p;
  return (int)p;
}
// Local view: row v keeps, in stored order, its entries (columns < kc) whose
// target lies in v's own group; the rest of the row is padding.  The exact
// pipeline on this view computes U_i MST_i,local (no edge joins two groups).
__global__ void k_local_view(const int32_t* __restrict__ nbr, const float* __restrict__ dist, int64_t n, int32_t ld,
                             int32_t kc, int P, int32_t* __restrict__ lnbr, float* __restrict__ ldist) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int pv = part_of(v, n, P);
    const int32_t* nr = nbr + v * ld;
    const float* dr = dist + v * ld;
    int32_t* on = lnbr + v * ld;
    float* od = ldist + v * ld;
    int o = 0;
    for (int c = 0; c < kc; ++c) {
      const int32_t J = nr[c];
      if (J >= 0 && J < n && part_of(J, n, P) == pv) {
        on[o] = J;
        od[o] = dr[c];
        ++o;
      }
    }
    for (; o < ld; ++o) {
      on[o] = -1;
      od[o] = __int_as_float(0x7f800000);
    }
  }
}
// E_cut: candidate entries of core rows whose target is a core point of another
// group, as survivors between local components (comp = dense local ids).
__global__ void k_cut_edges(const int32_t* __restrict__ nbr, const float* __restrict__ dist, int64_t n, int32_t ld,
                            int32_t kc, float eps, int P, const uint32_t* __restrict__ bits,
                            const int32_t* __restrict__ comp, HEdge* __restrict__ out, uint32_t cap,
                            uint32_t* __restrict__ n_out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    if (!is_core(bits, v)) continue;
    const int pv = part_of(v, n, P);
    const int32_t cv = comp[v];
    for (int c = 0; c < kc; ++c) {
      const float w = dist[v * ld + c];
      if (!(w <= eps)) break;
      const int64_t J = nbr[v * ld + c];
      if (J < 0 || J >= n || J == v || !is_core(bits, J) || part_of(J, n, P) == pv) continue;
      const uint32_t s = atomicAdd(n_out, 1u);
      if (s >= cap) atomicOr(n_out + 1, 1u);  // sticky overflow flag (the count could wrap)
      if (s < cap) {
        HEdge h;
        h.key = pack_key(mono_bits(w), (uint32_t)min(v, J));
        h.b = (uint32_t)max(v, J);
        h.x = cv;
        h.y = comp[J];
        h.pad = 0;
        out[s] = h;
      }
    }
  }
}

// heavy phase, per round: x = hcomp[e.x], y = hcomp[e.y]; intra -> dropped for
// good; else offer the key to both components (undirected)
__global__ void k_hedge_offer(const HEdge* __restrict__ E, uint32_t n, const int32_t* __restrict__ hcomp,
                              unsigned long long* __restrict__ Kc, uint8_t* __restrict__ keep) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const HEdge e = E[s];
    const int32_t x = gat(hcomp + e.x), y = gat(hcomp + e.y);
    const bool live = x != y;
    keep[s] = live;
    if (live) {
      min_offer(Kc + x, (unsigned long long)e.key);
      min_offer(Kc + y, (unsigned long long)e.key);
    }
  }
}

__global__ void k_hedge_tie(const HEdge* __restrict__ E, uint32_t n, const int32_t* __restrict__ hcomp,
                            const uint64_t* __restrict__ Kc, uint32_t* __restrict__ Bc) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const HEdge e = E[s];
    const int32_t x = gat(hcomp + e.x), y = gat(hcomp + e.y);
    if (e.key == gat(Kc + x)) atomicMin(Bc + x, e.b);
    if (e.key == gat(Kc + y)) atomicMin(Bc + y, e.b);
  }
}

// heavy-phase hook: the component of vertex u is hcomp[compL[u]]
__global__ void k_hook_h(int64_t C, const uint64_t* __restrict__ Kc, const uint32_t* __restrict__ Bc,
                         const int32_t* __restrict__ compL, const int32_t* __restrict__ hcomp,
                         int32_t* __restrict__ parent, uint64_t* __restrict__ e_key, float* __restrict__ e_w,
                         int64_t e_cap, RoundCounters* __restrict__ ctr) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < C; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = base + threadIdx.x;
    bool emit = false, offered = false;
    uint32_t a = 0, b = 0, wb = 0;
    if (c < C) {
      const uint64_t K = Kc[c];
      int32_t p = (int32_t)c;
      if (K != kSent) {
        offered = true;
        a = (uint32_t)K;
        b = Bc[c];
        wb = (uint32_t)(K >> 32);
        const int32_t ca = gat(hcomp + gat(compL + a));
        const int32_t t = ca == (int32_t)c ? gat(hcomp + gat(compL + b)) : ca;
        KDB_DCHECK(t >= 0 && t < C, 16u);
        const bool mutual = gat(Kc + t) == K && gat(Bc + t) == b;
        if (!(mutual && c < t)) {
          p = t;
          emit = true;
        }
      }
      parent[c] = p;
    }
    block_count(&ctr->offered, offered);
    block_count(&ctr->hooks, emit);
    const uint32_t slot = block_reserve(&ctr->msf_count, emit);
    if (emit && (int64_t)slot < e_cap) {
      e_key[slot] = ((uint64_t)b << 32) | wb;
      reinterpret_cast<uint32_t*>(e_w)[slot] = a;
    }
  }
}

__global__ void k_iota(int32_t* __restrict__ p, int64_t n) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    p[c] = (int32_t)c;
}

// hcomp[c] = map[hcomp[c]] over the light components
__global__ void k_relabel_h(int64_t n, int32_t* __restrict__ hcomp, const int32_t* __restrict__ map) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    hcomp[c] = gat(map + hcomp[c]);
}

