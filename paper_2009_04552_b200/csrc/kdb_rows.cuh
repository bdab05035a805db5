// kdb_rows.cuh -- core mark, initial state, in-edge lists and the Boruvka round kernels
// Part of kdb.cu's single translation unit: included inside its anonymous
// namespace, after kdb.cu's helpers; not a standalone header.
#pragma once

// ============================================================================
// a1: core marking
// ============================================================================
// One thread per 32-bit word of core flags: 32 independent loads of
// D[v][M-1] in flight, the word is stored whole (atomicOr only for the
// partial words at this rank's range ends; the caller zeroed the bits).
__global__ void k_core_mark(const float* __restrict__ dist, int64_t n_rows, int32_t k, int32_t M,
                            float eps, int64_t row_begin, uint32_t* __restrict__ bits) {
  const int64_t r_end = row_begin + n_rows;
  const int64_t w0 = row_begin >> 5, w1 = (r_end + 31) >> 5;
  for (int64_t wd = w0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; wd < w1;
       wd += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v0 = wd << 5;
    float d[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t v = v0 + j;
      d[j] = (v >= row_begin && v < r_end) ? __ldcs(dist + (v - row_begin) * k + (M - 1))
                                            : __int_as_float(0x7f800000);
    }
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) word |= (d[j] <= eps ? 1u : 0u) << j;
    if (v0 >= row_begin && v0 + 32 <= r_end)
      bits[wd] = word;
    else if (word)
      atomicOr(bits + wd, word);
  }
}

// ============================================================================
// a2: initial state
// ============================================================================
__global__ void k_popc_words(const uint32_t* __restrict__ bits, int64_t nwords, uint32_t* out) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x)
    out[w] = __popc(bits[w]);
}

// comp[v] = rank of v among core points (dense id) or -1; cmin[comp] = v
__global__ void k_init_comp(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ woff,
                            int64_t N, int32_t* __restrict__ comp, int32_t* __restrict__ cmin) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t word = bits[v >> 5];
    if ((word >> (v & 31)) & 1u) {
      const int32_t c = (int32_t)(woff[v >> 5] + __popc(word & ((1u << (v & 31)) - 1u)));
      comp[v] = c;
      cmin[c] = (int32_t)v;
    } else {
      comp[v] = -1;
    }
  }
}

__global__ void k_fill_comp_arrays(int64_t C, uint64_t* __restrict__ Kc, uint32_t* __restrict__ Bc,
                                   uint32_t* __restrict__ kmin, const int64_t* __restrict__ Cp = nullptr,
                                   ulonglong2* __restrict__ KB = nullptr) {
  if (Cp) C = *Cp;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    if (KB) {  // one rank, CAS offers: (key, b << 32 | target) words only
      KB[c] = make_ulonglong2(kSent, ~0ull);
      continue;
    }
    Kc[c] = kSent;
    Bc[c] = kSentB;
    if (kmin) kmin[c] = kInfBits;
  }
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Active rows and offers.  The scan position L[i] travels with
// the row id: one coalesced 8-byte record per live row.  Every entry before h is
// dead for good -- not a candidate, or intra-component (components only merge).
struct Rec {
  int32_t v;  // global row id
  int32_t h;  // head
};
// one row's (or in-list's) minimum leaving edge: its component, the key's b, the key
struct Offer {
  int32_t c;
  uint32_t b;
  uint64_t key;
};

// local rows: certificate bound kth'(v) into kmin[comp v] (exact mode); the
// active list holds the core rows whose first entry is within eps (a row
// starting beyond it offers nothing, ever).  comp[v] >= 0 <=> v is core.
__global__ void k_init_rows(const float* __restrict__ dist, int64_t n_rows, int32_t ld, int32_t k, float eps,
                            int64_t row_begin, const int32_t* __restrict__ comp, uint32_t* __restrict__ kmin,
                            Rec* __restrict__ act, uint32_t* __restrict__ n_act) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_rows; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = row_begin + i;
    bool want = false;
    if (i < n_rows) {
      const int32_t cv = comp[v];
      if (cv >= 0) {
        want = __ldcs(dist + i * ld) <= eps;
        if (kmin) {
          const float kth = __ldcs(dist + i * ld + (k - 1));
          kmin[cv] = (kth <= eps) ? mono_bits(kth) : kInfBits;
        }
      }
    }
    const uint32_t slot = block_reserve(n_act, want);
    if (want) act[slot] = Rec{(int32_t)v, 0};
  }
}

// ============================================================================
// general mode: in-edge lists (transpose of local candidate entries)
// ============================================================================
__global__ void k_in_count(const int32_t* __restrict__ nbr, const float* __restrict__ dist,
                           int64_t n_rows, int32_t ld, int32_t k, float eps, int64_t row_begin, int64_t N,
                           const uint32_t* __restrict__ bits, unsigned long long* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = row_begin + i;
    if (!is_core(bits, v)) continue;
    for (int32_t c = 0; c < k; ++c) {
      const float w = __ldg(dist + i * ld + c);
      if (!(w <= eps)) break;
      const int64_t J = __ldg(nbr + i * ld + c);
      if (J < 0 || J >= N || J == v || !is_core(bits, J)) continue;
      atomicAdd(cnt + J, 1ull);
    }
  }
}

__global__ void k_in_fill(const int32_t* __restrict__ nbr, const float* __restrict__ dist,
                          int64_t n_rows, int32_t ld, int32_t k, float eps, int64_t row_begin, int64_t N,
                          const uint32_t* __restrict__ bits, unsigned long long* __restrict__ cursor,
                          int32_t* __restrict__ in_src, float* __restrict__ in_w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = row_begin + i;
    if (!is_core(bits, v)) continue;
    for (int32_t c = 0; c < k; ++c) {
      const float w = __ldg(dist + i * ld + c);
      if (!(w <= eps)) break;
      const int64_t J = __ldg(nbr + i * ld + c);
      if (J < 0 || J >= N || J == v || !is_core(bits, J)) continue;
      const unsigned long long s = atomicAdd(cursor + J, 1ull);
      in_src[s] = (int32_t)v;
      in_w[s] = w;
    }
  }
}

// in_len[t] = count, in-active list = targets with in-edges
__global__ void k_in_finish(const unsigned long long* __restrict__ off, int64_t N,
                            int32_t* __restrict__ in_len, int32_t* __restrict__ in_active,
                            uint32_t* __restrict__ n_in_active) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < N;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = base + threadIdx.x;
    bool want = false;
    if (t < N) {
      const int32_t len = (int32_t)(off[t + 1] - off[t]);
      in_len[t] = len;
      want = len > 0;
    }
    const uint32_t slot = block_reserve(n_in_active, want);
    if (want) in_active[slot] = (int32_t)t;
  }
}


// ============================================================================
// a3: per-vertex minimum leaving entry (rows)
// ============================================================================
// For vertex v the incident edges of its row are ordered, under O1 with v fixed,
// by (mono(w), far id) (reading #6).  Rows are sorted by w, so the first entry
// at/after the head whose far endpoint lies in another component opens the
// minimum group; equal-weight entries after it may carry a smaller far id and
// are examined too.  The head only passes entries that can never leave again.
// comp[J] < 0 marks non-core J (not a candidate); J == v gives comp[J] == comp[v].
template <bool VEC>
__device__ __forceinline__ void load_chunk(const int32_t* nr, const float* dr, int c0, int k, int32_t (&J)[4],
                                           float (&w)[4]) {
  if (VEC) {  // row stride % 4 == 0: an aligned 4-chunk never straddles the row end (entries
              // at or beyond the candidate bound k are ignored by the callers)
    const int4 j4 = __ldcs(reinterpret_cast<const int4*>(nr + c0));
    const float4 w4 = __ldcs(reinterpret_cast<const float4*>(dr + c0));
    J[0] = j4.x; J[1] = j4.y; J[2] = j4.z; J[3] = j4.w;
    w[0] = w4.x; w[1] = w4.y; w[2] = w4.z; w[3] = w4.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool in = c0 + j < k;
      J[j] = in ? __ldcs(nr + c0 + j) : -1;
      w[j] = in ? __ldcs(dr + c0 + j) : __int_as_float(0x7f800000);
    }
  }
}

#ifndef KDB_SLIM
#define KDB_SLIM 1  // 1 (default) = loop-carried scan flags in full registers instead of packed bytes (54 -> 15 PRMT
#endif              // in k_light_round, C4 light rounds 10.17 -> 10.08 ms); A/B builds libkdb_slim<n>.so: 0 = bool flags;
                    // 2 = + scan_ell's tail out of line (11.9 ms: the call pins the scan state); 3 = + record loop not
                    // unrolled (12.1 ms)
#if KDB_SLIM
typedef int scan_flag_t;
#else
typedef bool scan_flag_t;
#endif
struct RowScan {
  scan_flag_t found;
  int h;          // new head: the first leaving entry, or k when exhausted
  uint64_t best;  // minimum key of the group
  uint32_t bestb;
  int32_t bestc;  // component of the best entry's far endpoint
  int bidx;       // scan_ell: ELL column of the best entry (-1: past the ELL); else unset
  bool cont = false;  // scan_ell<ONE>: nothing found in this chunk, the row goes on at column h
};

// Local-first phase (multi-rank exact mode): a rank contracts
// its own rows before any exchange.  Component ids are then LOCAL (dense over
// the rank's core rows) and an entry whose far endpoint lies outside the
// rank's rows [lo, hi) is a leaving edge to a component this rank cannot see:
// its component reads as kRemote (>= 0, so it leaves; never a local id).
// bits == nullptr: the global view (every id is local, dense ids global).
constexpr int32_t kRemote = 0x7fffffff;
// Light ELL layout: kW/4 chunks of 32 B ((J, w bits) x 4) per row.
// 0 (default): row-major 128-B rows.  KDB_ELL_PLANES=1: plane p holds chunk p
// of every row -- a round reading one chunk per row in row order uses whole
// 128-B lines (round 2 of C4: 4.3 GB of DRAM instead of 9.3 GB), but the
// light rounds took 12.58 ms against 11.77 ms in a same-box A/B: a row-major
// line brings the row's next chunks along for the scans that continue.
#ifndef KDB_ELL_PLANES
#define KDB_ELL_PLANES 0
#endif
__host__ __device__ __forceinline__ int64_t ell_row(int64_t i) { return KDB_ELL_PLANES ? 2 * i : 8 * i; }  // 8 = kW / 2 int4 per row
__host__ __device__ __forceinline__ int64_t ell_ps(int64_t n_rows) { return KDB_ELL_PLANES ? 2 * n_rows : 2; }

struct LocalView {
  int64_t lo = 0, hi = 0;
  const uint32_t* bits = nullptr;
  uint64_t pol = 0;  // L2 cache policy for the component gathers (0: default)
  int l1 = 0;        // component gathers through L1 (read-only path): rows of spatially ordered ids
  // global phase of the local-first scheme: comp[] holds the transition ids
  // for the whole phase and gmap[transition id] the current component, so a
  // round relabels the C_G-sized map instead of all N vertices
  const int32_t* gmap = nullptr;
};
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int32_t gat_hint(const int32_t* p, uint64_t pol) {
  int32_t r;
  asm volatile("ld.global.cg.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
// component of far endpoint J (< 0: not a candidate, i.e. non-core); direct:
// singleton components whose dense id is the vertex's position in the view
__device__ __forceinline__ int32_t comp_of(const int32_t* __restrict__ comp, int64_t J, bool direct,
                                           const LocalView& lv) {
  if (lv.bits && (J < lv.lo || J >= lv.hi)) return is_core(lv.bits, J) ? kRemote : -1;
  if (direct) return (int32_t)(J - lv.lo);
  if (lv.gmap) {
    const int32_t c = gat(comp + J);
    return c >= 0 ? gat(lv.gmap + c) : c;
  }
  if (lv.l1) return __ldg(comp + J);  // comp is read-only while a round runs (k_relabel writes it)
  return lv.pol ? gat_hint(comp + J, lv.pol) : gat(comp + J);
}
// The gather with its view fixed at compile time (the later light rounds of
// the one-view case: no rank window, no global map -- ncu showed the runtime
// dispatch above as ~20 of the ~80 instructions per scanned entry).
// GM 0: runtime view (comp_of); 1: read-only path (L1); 2: L2 policy hint.
enum { kGmRuntime = 0, kGmL1 = 1, kGmHint = 2 };
template <int GM>
__device__ __forceinline__ int32_t comp_of_m(const int32_t* __restrict__ comp, int64_t J, bool direct,
                                             const LocalView& lv) {
  if (GM == kGmL1) return __ldg(comp + J);
  if (GM == kGmHint) return gat_hint(comp + J, lv.pol);
  return comp_of(comp, J, direct, lv);
}

// Scan row (nr, dr) of vertex v (component cv) from head h.  direct: singleton
// components (round 1, exact mode) -- every candidate leaves; with all_core the
// dense component id of a vertex is the vertex itself (no gathers at all).
template <bool VEC, bool DIRECT>
__device__ __forceinline__ RowScan scan_row(const int32_t* __restrict__ nr, const float* __restrict__ dr, int k,
                                            float eps, int32_t v, int32_t cv, int h, int64_t N,
                                            const int32_t* __restrict__ comp, int all_core,
                                            unsigned long long& reads, const LocalView lv = LocalView{}) {
  RowScan r{false, k, kSent, kSentB, -1};
  float wstar = 0.f;
  int c0 = h & ~3;
  bool done = false;
  while (!done && c0 < k) {
    int32_t J[4];
    float w[4];
    load_chunk<VEC>(nr, dr, c0, k, J, w);
    int32_t cj[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int idx = c0 + j;
      const bool cand = idx >= h && idx < k && w[j] <= eps && J[j] >= 0 && J[j] < N && J[j] != v;
      cj[j] = cand ? comp_of(comp, J[j], DIRECT && all_core, lv) : -1;
    }
    reads += (unsigned long long)(min(c0 + 4, k) - max(c0, h));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int idx = c0 + j;
      if (done || idx < h || idx >= k) continue;
      const bool leaving = cj[j] >= 0 && (DIRECT || cj[j] != cv);
      if (!r.found) {
        if (!(w[j] <= eps)) { r.h = k; done = true; continue; }  // sorted: nothing left
        if (!leaving) { h = idx + 1; continue; }                   // dead entry
        r.found = true;
        r.h = idx;
        wstar = w[j];
        r.best = pack_key(mono_bits(w[j]), (uint32_t)min(v, J[j]));
        r.bestb = (uint32_t)max(v, J[j]);
        r.bestc = cj[j];
      } else {
        if (w[j] != wstar) { done = true; continue; }
        if (!leaving) continue;
        const uint64_t kk = pack_key(mono_bits(w[j]), (uint32_t)min(v, J[j]));
        const uint32_t bb = (uint32_t)max(v, J[j]);
        if (kk < r.best || (kk == r.best && bb < r.bestb)) { r.best = kk; r.bestb = bb; r.bestc = cj[j]; }
      }
    }
    c0 += 4;
  }
  if (!r.found) r.h = k;
  return r;
}

// Round 1 with singleton components (exact mode): the row's first candidate
// group IS its component's minimum -- no atomics and no tie pass; the owner
// writes Kc, Bc and the hook target directly.  Rows that offered stay active.
template <bool VEC>
__global__ void __launch_bounds__(256) k_offer_first(const int32_t* __restrict__ nbr, const float* __restrict__ dist,
                                                     int32_t ld, int32_t k, float eps, int64_t row_begin, int64_t N,
                                                     const int32_t* __restrict__ comp, int all_core,
                                                     const Rec* __restrict__ act, uint32_t n_in,
                                                     Rec* __restrict__ act_out, uint32_t* __restrict__ n_out,
                                                     uint64_t* __restrict__ Kc, uint32_t* __restrict__ Bc,
                                                     int32_t* __restrict__ tgt, unsigned long long* __restrict__ n_entries, const uint32_t* __restrict__ n_in_p = nullptr) {
  if (n_in_p) n_in = *n_in_p;
  unsigned long long reads = 0;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n_in; base += gridDim.x * blockDim.x) {
    const uint32_t s = base + threadIdx.x;
    RowScan r{false, 0, kSent, kSentB, -1};
    int32_t v = -1;
    if (s < n_in) {
      const int2 a2 = __ldcs(reinterpret_cast<const int2*>(act + s));
      const Rec a{a2.x, a2.y};
      v = a.v;
      const int64_t i = (int64_t)v - row_begin;
      r = scan_row<VEC, true>(nbr + i * ld, dist + i * ld, k, eps, v, -1, a.h, N, comp, all_core, reads);
      if (r.found) {
        const int32_t cv = all_core ? v : gat(comp + v);
        Kc[cv] = r.best;
        Bc[cv] = r.bestb;
        tgt[cv] = r.bestc;
      }
    }
    const uint32_t slot = block_reserve(n_out, r.found);
    if (r.found) act_out[slot] = Rec{v, r.h};
  }
  for (int o = 16; o > 0; o >>= 1) reads += __shfl_xor_sync(0xffffffffu, reads, o);
  if ((threadIdx.x & 31) == 0 && reads) atomicAdd(n_entries, reads);
}

// Later rounds: one thread per live row; the offer goes to Kc[comp v] by a
// 64-bit atomicMin (Alg. 3 pwrite, reading #7) and, with the
// row's next record, to the same slot of the offer list (for the tie pass).
template <bool VEC>
__global__ void __launch_bounds__(256) k_offer_round(const int32_t* __restrict__ nbr, const float* __restrict__ dist,
                                                     int32_t ld, int32_t k, float eps, int64_t row_begin, int64_t N,
                                                     const int32_t* __restrict__ comp, const Rec* __restrict__ act,
                                                     uint32_t n_in, Rec* __restrict__ act_out,
                                                     uint32_t* __restrict__ n_out, Offer* __restrict__ offers,
                                                     unsigned long long* __restrict__ Kc,
                                                     unsigned long long* __restrict__ n_entries, const uint32_t* __restrict__ n_in_p = nullptr,
                                                     int precheck = 0) {
  if (n_in_p) n_in = *n_in_p;
  unsigned long long reads = 0;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n_in; base += gridDim.x * blockDim.x) {
    const uint32_t s = base + threadIdx.x;
    RowScan r{false, 0, kSent, kSentB, -1};
    int32_t v = -1, cv = -1;
    if (s < n_in) {
      const int2 a2 = __ldcs(reinterpret_cast<const int2*>(act + s));
      const Rec a{a2.x, a2.y};
      v = a.v;
      cv = gat(comp + v);
      const int64_t i = (int64_t)v - row_begin;
      r = scan_row<VEC, false>(nbr + i * ld, dist + i * ld, k, eps, v, cv, a.h, N, comp, 0, reads);
      if (r.found) {
        if (precheck) min_offer(Kc + cv, (unsigned long long)r.best);
        else atomicMin(Kc + cv, (unsigned long long)r.best);
      }
    }
    const uint32_t slot = block_reserve(n_out, r.found);
    if (r.found) {
      act_out[slot] = Rec{v, r.h};
      offers[slot] = Offer{cv, r.bestb, r.best};
    }
  }
  for (int o = 16; o > 0; o >>= 1) reads += __shfl_xor_sync(0xffffffffu, reads, o);
  if ((threadIdx.x & 31) == 0 && reads) atomicAdd(n_entries, reads);
}

// ---------------------------------------------------------------------------
// Light ELL.  A random visit of a 400-byte-strided graph row is expensive
// (scattered sectors, HBM row activations), so the first kW columns of every
// core row are copied ONCE into a dense, 128-byte-aligned ELL of (J, w bits)
// pairs and every Boruvka round reads that instead.  Rows whose candidate
// prefix (w <= eps_run) runs past column kW continue in the graph row itself.
constexpr int kW = 16;
static_assert(kW == 16, "ell_row() assumes kW / 2 == 8 int4 per row");

// one 32-byte streaming load (evict-first: LDG.E.EF.ENL2.256) -- a light-ELL
// chunk is read once per round; keep L2 for the component gathers
__device__ __forceinline__ void ld256cs(const int4* p, int4& a, int4& b) {
  asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

// one 32-byte load (sm_100: LDG.E.ENL2.256); p must be 32-byte aligned
__device__ __forceinline__ void ld256(const int4* p, int4& a, int4& b) {
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

// records per chunk of the ordered row kernels (see k_light_first)
constexpr int kChunk = 1024;

// one thread per row: 4 x (int4 + float4) loads in flight, 8 x int4 stores.
// Exact mode also writes the certificate bound kth'(v) into kmin[comp v]; kth
// is only loaded when the ELL row is entirely within eps (else kth > eps).
// Rows are taken in ordered chunks; the initial list keeps row order.
template <bool VEC, bool A32>
__global__ void __launch_bounds__(256) k_light_ell(const int32_t* __restrict__ nbr, const float* __restrict__ dist,
                                                   int64_t n_rows, int32_t ld, int32_t k, float eps, int64_t row_begin,
                                                   const int32_t* __restrict__ comp, uint32_t* __restrict__ kmin,
                                                   int4* __restrict__ LE, Rec* __restrict__ act,
                                                   uint32_t* __restrict__ n_act, uint32_t* __restrict__ grab,
                                                   int direct, int all_core, int64_t N, uint64_t* __restrict__ Kc,
                                                   uint32_t* __restrict__ Bc, int32_t* __restrict__ tgt,
                                                   int4* __restrict__ rec1, uint32_t* __restrict__ n_deep,
                                                   const LocalView lv = LocalView{}, int skip1 = 1,
                                                   int chunk = kChunk, uint32_t* __restrict__ kthL = nullptr) {
  __shared__ __align__(16) Rec s_rec[kChunk];
  __shared__ uint32_t s_n, s_chunk, s_base;
  uint32_t deep = 0;  // rows whose kW ELL entries are all within eps (their scans go past the first chunk)
  uint32_t local = 0;  // rows whose nearest neighbour has a nearby id (RoundCounters::n_local)
  for (;;) {
    if (threadIdx.x == 0) { s_chunk = atomicAdd(grab, 1u); s_n = 0; }
    __syncthreads();
    const int64_t base = (int64_t)s_chunk * chunk;
    if (base >= n_rows) break;
    for (int t = 0; t < chunk; t += 256) {
      const int64_t i = base + t + threadIdx.x;
      if (i >= n_rows) continue;
      const int64_t v = row_begin + i;
      const int32_t cv = comp[v];
      // kthL != null: the ELL (and each row's certificate bound) is kept for the
      // next call on the same graph (an eps sweep, KDB_GRAPH_REUSE): non-core
      // rows get theirs too -- another eps may make them core
      if (cv < 0 && !kthL) continue;
      const int32_t* nr = nbr + i * ld;
      const float* dr = dist + i * ld;
      int32_t J[kW];
      float w[kW];
      if (VEC && A32) {
        // whole 32-byte sectors (LDG.256): a row starts at a 32-B boundary or
        // 16 B past one (ld % 8 == 4), so 2 or 3 sectors cover its first kW
        // entries -- one request per sector instead of one per 16-B half
        const int sh = (int)((i * ld) & 7);  // 0 or 4
        int4 a0, a1, a2, a3, a4, a5, b0, b1, b2, b3, b4, b5;
        const int4* pj = reinterpret_cast<const int4*>(nr - sh);
        const int4* pd = reinterpret_cast<const int4*>(dr - sh);
        ld256(pj, a0, a1);
        ld256(pj + 2, a2, a3);
        ld256(pd, b0, b1);
        ld256(pd + 2, b2, b3);
        if (sh) {
          ld256(pj + 4, a4, a5);
          ld256(pd + 4, b4, b5);
        } else {
          a4 = a5 = b4 = b5 = make_int4(0, 0, 0, 0);
        }
        const int32_t SJ[24] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w,
                                a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, a4.z, a4.w, a5.x, a5.y, a5.z, a5.w};
        const int32_t SW[24] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w,
                                b3.x, b3.y, b3.z, b3.w, b4.x, b4.y, b4.z, b4.w, b5.x, b5.y, b5.z, b5.w};
#pragma unroll
        for (int c = 0; c < kW; ++c) {
          J[c] = sh ? SJ[c + 4] : SJ[c];
          w[c] = __int_as_float(sh ? SW[c + 4] : SW[c]);
        }
      } else if (VEC && ld >= kW) {
#pragma unroll
        for (int q = 0; q < kW / 4; ++q) {
          // L1-allocating loads: the two 16-B halves of a sector are separate
          // instructions; the second must hit L1, not re-request the sector
          const int4 j4 = __ldg(reinterpret_cast<const int4*>(nr + 4 * q));
          const float4 w4 = __ldg(reinterpret_cast<const float4*>(dr + 4 * q));
          J[4 * q] = j4.x; J[4 * q + 1] = j4.y; J[4 * q + 2] = j4.z; J[4 * q + 3] = j4.w;
          w[4 * q] = w4.x; w[4 * q + 1] = w4.y; w[4 * q + 2] = w4.z; w[4 * q + 3] = w4.w;
        }
      } else {
#pragma unroll
        for (int c = 0; c < kW; ++c) {
          J[c] = c < k ? __ldg(nr + c) : -1;
          w[c] = c < k ? __ldg(dr + c) : __int_as_float(0x7f800000);
        }
      }
      if (VEC && k < kW) {  // edge_cols < kW: columns >= k are not candidates (padding)
#pragma unroll
        for (int c = 0; c < kW; ++c)
          if (c >= k) { J[c] = -1; w[c] = __int_as_float(0x7f800000); }
      }
      // kth = D[v][k-1] >= D[v][kW-1]: only needed (exact-mode certificate) when
      // that is within eps_run
      uint32_t kb = kInfBits;
      if (kmin) {
        float kth = __int_as_float(0x7f800000);
        if (k <= kW || w[kW - 1] <= eps) kth = __ldcs(dr + (k - 1));
        kb = (kth <= eps) ? mono_bits(kth) : kInfBits;
        if (cv >= 0) kmin[cv] = kb;
        if (kthL) kthL[i] = kb;
      }
      deep += w[kW - 1] <= eps;
      local += (uint32_t)(J[0] >= 0 && (uint32_t)abs((int64_t)J[0] - v) < 65536u);
      // chunk p (entries 4p..4p+3, 32 B) of row i: ell_chunk (planes or rows)
      int4* o = LE + ell_row(i);
#pragma unroll
      for (int q = 0; q < kW / 2; ++q)
        __stcs(o + (int64_t)(q >> 1) * ell_ps(n_rows) + (q & 1),
               make_int4(J[2 * q], __float_as_int(w[2 * q]), J[2 * q + 1], __float_as_int(w[2 * q + 1])));
      if (cv < 0) continue;
      if (!direct) {
        if (w[0] <= eps) s_rec[atomicAdd(&s_n, 1u)] = Rec{(int32_t)v, 0};
        continue;
      }
      // Round 1 fused (exact mode, singleton components): the row's first
      // candidate group, from the registers, is its component's minimum (see
      // k_light_first); the list written is round 1's OUTPUT (rows that offered).
      RowScan r{false, (int)k, kSent, kSentB, -1};
      float wstar = 0.f;
      bool done = false;
      int bidx = -1;  // column of the row's minimum
#pragma unroll
      for (int c = 0; c < kW; ++c) {
        if (done || c >= k) continue;
        const int32_t Jc = J[c];
        if (!r.found) {
          if (!(w[c] <= eps)) { done = true; continue; }  // sorted: no candidate at all
          if (Jc < 0 || Jc >= N || Jc == v) continue;
          const int32_t cc = comp_of(comp, Jc, all_core, lv);
          if (cc < 0) continue;
          r.found = true;
          bidx = c;
          r.h = c;
          wstar = w[c];
          r.best = pack_key(mono_bits(w[c]), (uint32_t)min(v, (int64_t)Jc));
          r.bestb = (uint32_t)max(v, (int64_t)Jc);
          r.bestc = cc;
        } else {
          if (w[c] != wstar) { done = true; continue; }
          if (Jc < 0 || Jc >= N || Jc == v) continue;
          const int32_t cc = comp_of(comp, Jc, all_core, lv);
          if (cc < 0) continue;
          const uint64_t kk = pack_key(mono_bits(w[c]), (uint32_t)min(v, (int64_t)Jc));
          const uint32_t bb = (uint32_t)max(v, (int64_t)Jc);
          if (kk < r.best || (kk == r.best && bb < r.bestb)) { r.best = kk; r.bestb = bb; r.bestc = cc; bidx = c; }
        }
      }
      if (!done && k > kW) {  // the search or the tie group runs past the ELL: scan the row in place
        unsigned long long rd = 0;
        r = scan_row<false, true>(nr, dr, k, eps, (int32_t)v, -1, 0, N, comp, all_core, rd, lv);
        bidx = -1;
      }
      // The singleton {v} hooks along its minimum when that is certified (and,
      // in a local-first phase, stays inside the rank): then the entry at the
      // head is intra from round 2 on and the round-2 scan need not gather it
      // (every row's first visit would otherwise re-read its nearest neighbour).
      const bool skip_head = skip1 && r.found && bidx == r.h && r.bestc != kRemote && (uint32_t)(r.best >> 32) < kb;
      if (rec1) {  // single rank: one packed record per component for k_hook<true>
        __stcg(rec1 + cv, make_int4((int)(uint32_t)r.best, (int)(uint32_t)(r.best >> 32), (int)r.bestb, (int)kb));
        if (r.found) tgt[cv] = r.bestc;
      } else if (r.found) {
        Kc[cv] = r.best;
        Bc[cv] = r.bestb;
        tgt[cv] = r.bestc;
      }
      if (r.found) s_rec[atomicAdd(&s_n, 1u)] = Rec{(int32_t)v, skip_head ? r.h + 1 : r.h};
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_n ? atomicAdd(n_act, s_n) : 0u;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < s_n; j += blockDim.x) act[s_base + j] = s_rec[j];
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) {
    deep += __shfl_xor_sync(0xffffffffu, deep, o);
    local += __shfl_xor_sync(0xffffffffu, local, o);
  }
  if ((threadIdx.x & 31) == 0 && deep) atomicAdd(n_deep, deep);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(n_deep + 1, local);  // RoundCounters::n_local
}



// eps sweep on an unchanged graph (KDB_GRAPH_REUSE): the light ELL and each
// row's certificate bound were kept by the previous call (they depend on the
// graph and the light threshold, not on eps); only the core-dependent state
// is rebuilt: kmin per component and the active list (core rows whose first
// entry is within eps_run) -- round 1 then runs over the ELL (k_light_first).
__global__ void k_reuse_rows(const int4* __restrict__ LE, const uint32_t* __restrict__ kthL, int64_t n_rows,
                             int64_t row_begin, float eps, const int32_t* __restrict__ comp, uint32_t* __restrict__ kmin,
                             Rec* __restrict__ act, uint32_t* __restrict__ n_act, int4* __restrict__ rec1 = nullptr) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_rows; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool want = false;
    if (i < n_rows) {
      const int32_t cv = comp[row_begin + i];
      if (cv >= 0) {
        kmin[cv] = kthL[i];
        // packed round 1 (k_hook<true>) reads every component's record: the
        // sentinel with the certificate bound; k_light_first overwrites offers
        if (rec1) __stcg(rec1 + cv, make_int4(-1, -1, -1, (int)kthL[i]));
        want = __int_as_float(__ldcs(reinterpret_cast<const int*>(LE + ell_row(i)) + 1)) <= eps;
      }
    }
    const uint32_t slot = block_reserve(n_act, want);
    if (want) act[slot] = Rec{(int32_t)(row_begin + i), 0};
  }
}

// Scan row v (component cv) from head h: columns < kW from the ELL row, the
// rest (rare: a candidate prefix longer than kW) from the graph row.  DIRECT:
// singleton components (round 1, exact mode), every candidate leaves; with
// all_core a vertex's dense component id is the vertex itself (no gathers).
// GW: component gathers are issued GW entries at a time; once the minimum is
// found only entries of its weight (decided from the loaded w) are gathered,
// so a smaller GW trades memory-level parallelism for L2 sector traffic.
// The rare tail of scan_ell (the candidate prefix or the minimum's tie group runs
// past the kW ELL columns into the graph row), out of line under KDB_SLIM so the
// light-round kernels' hot loop stays small (2,768 SASS instructions with it inline;
// ncu: ~7% of stall samples are no_instruction).
template <bool DIRECT, int GM>
__device__ __noinline__ void scan_ell_tail(RowScan& r, uint32_t wstar, const int32_t* __restrict__ nr,
                                           const float* __restrict__ dr, int k, float eps, int32_t v, int32_t cv, int h,
                                           int64_t N, const int32_t* __restrict__ comp, int all_core,
                                           unsigned long long& reads, const LocalView& lv) {
  if (!r.found) {
    r = scan_row<false, DIRECT>(nr, dr, k, eps, v, cv, max(h, kW), N, comp, all_core, reads, lv);
    r.bidx = -1;
    return;
  }
  for (int c = kW; c < k; ++c) {
    const float wc = __ldcg(dr + c);
    if (mono_bits(wc) != wstar || !(wc <= eps)) break;
    const int32_t Jc = __ldcg(nr + c);
    ++reads;
    if (Jc < 0 || Jc >= N || Jc == v) continue;
    const int32_t cc = comp_of_m<GM>(comp, Jc, DIRECT && all_core, lv);
    if (cc < 0 || (!DIRECT && cc == cv)) continue;
    const uint64_t kk = pack_key(wstar, (uint32_t)min(v, Jc));
    const uint32_t bb = (uint32_t)max(v, Jc);
    if (kk < r.best || (kk == r.best && bb < r.bestb)) { r.best = kk; r.bestb = bb; r.bestc = cc; r.bidx = -1; }
  }
}

template <bool DIRECT, int GW = 4, bool PIPE = false, int GM = kGmRuntime, bool ONE = false>
__device__ __forceinline__ RowScan scan_ell(const int4* __restrict__ le, int64_t ps, const int32_t* __restrict__ nr,
                                            const float* __restrict__ dr, int k, float eps, int32_t v, int32_t cv,
                                            int h, int64_t N, const int32_t* __restrict__ comp, int all_core,
                                            unsigned long long& reads, const LocalView lv = LocalView{}) {
  RowScan r{false, k, kSent, kSentB, -1};
  uint32_t wstar = 0;
  const int kend = min(k, kW);
  int c0 = h & ~3;
  scan_flag_t done = false;
  // PIPE: the next chunk's load is issued with the current one, so a row whose
  // chunk holds no leaving entry does not wait a second load latency (chosen per
  // input: pays when many rows scan past their first chunk, see rows_phase)
  int4 q0, q1;
  if (PIPE && c0 < kend) ld256cs(le + (int64_t)(c0 >> 2) * ps, q0, q1);
  while (!done && c0 < kend) {
    int4 p0, p1;
    if (PIPE) {
      p0 = q0;
      p1 = q1;
      if (c0 + 4 < kend) ld256cs(le + (int64_t)((c0 + 4) >> 2) * ps, q0, q1);
    } else {
      ld256cs(le + (int64_t)(c0 >> 2) * ps, p0, p1);
    }
    const int32_t J[4] = {p0.x, p0.z, p1.x, p1.z};
    const float w[4] = {__int_as_float(p0.y), __int_as_float(p0.w), __int_as_float(p1.y), __int_as_float(p1.w)};
    reads += (unsigned long long)(min(c0 + 4, kend) - max(c0, h));
#pragma unroll
    for (int g0 = 0; g0 < 4; g0 += GW) {
    if (done) break;
    int32_t cj[4];
#pragma unroll
    for (int j = g0; j < g0 + GW; ++j) {
      const int idx = c0 + j;
      // (uint32_t)J < N: J >= 0 and J < N in one compare (N < 2^31, kdb_mst's check)
      bool cand = idx >= h && idx < kend && w[j] <= eps && (uint32_t)J[j] < (uint32_t)N && J[j] != v;
      if (GW < 4 && r.found && mono_bits(w[j]) != wstar) cand = false;  // past the tie group: no gather
      cj[j] = cand ? comp_of_m<GM>(comp, J[j], DIRECT && all_core, lv) : -1;
    }
#pragma unroll
    for (int j = g0; j < g0 + GW; ++j) {
      const int idx = c0 + j;
      if (done || idx < h || idx >= kend) continue;
      const bool leaving = cj[j] >= 0 && (DIRECT || cj[j] != cv);
      const uint32_t wb = mono_bits(w[j]);
      if (!r.found) {
        if (!(w[j] <= eps)) { r.h = k; done = true; continue; }  // sorted: nothing left
        if (!leaving) { h = idx + 1; continue; }                   // dead entry
        r.found = true;
        r.h = idx;
        wstar = wb;
        r.best = pack_key(wb, (uint32_t)min(v, J[j]));
        r.bestb = (uint32_t)max(v, J[j]);
        r.bestc = cj[j];
        r.bidx = idx;
      } else {
        if (wb != wstar) { done = true; continue; }
        if (!leaving) continue;
        const uint64_t kk = pack_key(wb, (uint32_t)min(v, J[j]));
        const uint32_t bb = (uint32_t)max(v, J[j]);
        if (kk < r.best || (kk == r.best && bb < r.bestb)) { r.best = kk; r.bestb = bb; r.bestc = cj[j]; r.bidx = idx; }
      }
    }
    }
    c0 += 4;
    // ONE (k_light_lvl): one chunk per visit unless a minimum's tie group runs on
    if (ONE && !done && !r.found && c0 < kend) { r.h = c0; r.cont = true; return r; }
  }
#if KDB_SLIM >= 2
  if (!done && k > kW) {
    const bool was_found = r.found;
    scan_ell_tail<DIRECT, GM>(r, wstar, nr, dr, k, eps, v, cv, h, N, comp, all_core, reads, lv);
    if (!was_found) return r;
  }
#else
  if (!done && k > kW) {
    // the candidate prefix (or the minimum's tie group) runs past the ELL
    if (!r.found) {
      RowScan t = scan_row<false, DIRECT>(nr, dr, k, eps, v, cv, max(h, kW), N, comp, all_core, reads, lv);
      t.bidx = -1;
      return t;
    }
    // continue the tie group of weight wstar in the graph row
    for (int c = kW; c < k; ++c) {
      const float wc = __ldcg(dr + c);
      if (mono_bits(wc) != wstar || !(wc <= eps)) break;
      const int32_t Jc = __ldcg(nr + c);
      ++reads;
      if (Jc < 0 || Jc >= N || Jc == v) continue;
      const int32_t cc = comp_of_m<GM>(comp, Jc, DIRECT && all_core, lv);
      if (cc < 0 || (!DIRECT && cc == cv)) continue;
      const uint64_t kk = pack_key(wstar, (uint32_t)min(v, Jc));
      const uint32_t bb = (uint32_t)max(v, Jc);
      if (kk < r.best || (kk == r.best && bb < r.bestb)) { r.best = kk; r.bestb = bb; r.bestc = cc; r.bidx = -1; }
    }
  }
#endif
  if (!r.found) r.h = k;
  return r;
}

// scan_ell<false, 4, false> for the later light rounds of the one-view case
// (GM != kGmRuntime), as straight-line selects instead of the per-entry branch
// ladder: ncu of round 3 (C4) showed ~80 warp instructions per scanned entry,
// half of them the ladder's divergent paths at 13-18 active lanes.  Same
// result: the first valid entry beyond eps ends a row with nothing found; dead
// entries (not leaving) before the first leaving one are passed over; the
// minimum is the first leaving entry and its tie group (equal weight bits)
// competes by (key, b); the first other weight ends the scan.  Only a row's
// final head matters here (r.h = the minimum's column, else k), so the dead
// prefix is not tracked entry by entry.
template <int GM, bool ONE = false>
__device__ __forceinline__ RowScan scan_ell_fast(const int4* __restrict__ le, int64_t ps,
                                                 const int32_t* __restrict__ nr, const float* __restrict__ dr, int k,
                                                 float eps, int32_t v, int32_t cv, int h, int64_t N,
                                                 const int32_t* __restrict__ comp, unsigned long long& reads,
                                                 const LocalView lv) {
  const int kend = min(k, kW);
  const uint32_t n32 = (uint32_t)N;  // N < 2^31 (kdb_mst's check): J >= 0 && J < N in one compare
  bool found = false, done = false;
  uint32_t wstar = 0;
  uint64_t best = kSent;
  uint32_t bestb = kSentB;
  int32_t bestc = -1;
  int fh = k;
  for (int c0 = h & ~3; c0 < kend; c0 += 4) {
    int4 p0, p1;
    ld256cs(le + (int64_t)(c0 >> 2) * ps, p0, p1);
    const int32_t J[4] = {p0.x, p0.z, p1.x, p1.z};
    const float w[4] = {__int_as_float(p0.y), __int_as_float(p0.w), __int_as_float(p1.y), __int_as_float(p1.w)};
    reads += (unsigned long long)(min(c0 + 4, kend) - max(c0, h));
    int32_t cj[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int idx = c0 + j;
      const bool cand = idx >= h && idx < kend && w[j] <= eps && (uint32_t)J[j] < n32 && J[j] != v;
      cj[j] = cand ? comp_of_m<GM>(comp, J[j], false, lv) : -1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int idx = c0 + j;
      const bool valid = idx >= h && idx < kend && !done;
      const bool in = w[j] <= eps;
      const bool leave = cj[j] >= 0 && cj[j] != cv;
      const uint32_t wb = mono_bits(w[j]);
      const uint64_t key = pack_key(wb, (uint32_t)min(v, J[j]));
      const uint32_t bb = (uint32_t)max(v, J[j]);
      const bool first = valid && !found && in && leave;
      const bool stop0 = valid && !found && !in;  // sorted: nothing left
      const bool eq = wb == wstar;
      const bool end = valid && found && !eq;     // past the minimum's tie group
      const bool better = valid && found && eq && leave && (key < best || (key == best && bb < bestb));
      const bool take = first || better;
      best = take ? key : best;
      bestb = take ? bb : bestb;
      bestc = take ? cj[j] : bestc;
      fh = first ? idx : fh;
      wstar = first ? wb : wstar;
      found = found || first;
      done = done || stop0 || end;
    }
    if (done) break;
    // ONE (k_light_pool): one chunk per visit unless a minimum's tie group runs on
    if (ONE && !found && c0 + 4 < kend) return RowScan{false, c0 + 4, best, bestb, bestc, -1, true};
  }
  if (!done && k > kW) {
    // the candidate prefix (or the minimum's tie group) runs past the ELL (rare)
    if (!found) return scan_row<false, false>(nr, dr, k, eps, v, cv, max(h, kW), N, comp, 0, reads, lv);
    for (int c = kW; c < k; ++c) {  // continue the tie group of weight wstar in the graph row
      const float wc = __ldcg(dr + c);
      if (mono_bits(wc) != wstar || !(wc <= eps)) break;
      const int32_t Jc = __ldcg(nr + c);
      ++reads;
      if (Jc < 0 || Jc >= N || Jc == v) continue;
      const int32_t cc = comp_of_m<GM>(comp, Jc, false, lv);
      if (cc < 0 || cc == cv) continue;
      const uint64_t kk = pack_key(wstar, (uint32_t)min(v, Jc));
      const uint32_t bb = (uint32_t)max(v, Jc);
      if (kk < best || (kk == best && bb < bestb)) { best = kk; bestb = bb; bestc = cc; }
    }
  }
  return RowScan{found, found ? fh : k, best, bestb, bestc, -1};
}

// scan_ell for the later light rounds (not DIRECT, all four gathers of a
// chunk at once, no pipelining) on 4-bit masks instead of a per-entry branch
// ladder: the dead prefix ends at the first valid entry that is beyond eps or
// leaving (ffs), the minimum's tie group is the run of equal weights after it
// (rows are sorted by weight), and keys are packed only for the minimum and its
// leaving ties.  Same result as scan_ell<false, 4, false> (parity-green), but
// measured slower (C4: 33.7 against 33.2 ms per step, same box): the mask
// bookkeeping costs more issue slots than the branches it replaces; off
// (KDB_LEAN=1 selects it).
__device__ __forceinline__ RowScan scan_ell_lean(const int4* __restrict__ le, int64_t ps,
                                                 const int32_t* __restrict__ nr, const float* __restrict__ dr, int k,
                                                 float eps, int32_t v, int32_t cv, int h, int64_t N,
                                                 const int32_t* __restrict__ comp, unsigned long long& reads,
                                                 const LocalView lv) {
  RowScan r{false, k, kSent, kSentB, -1};
  uint32_t wstar = 0;
  const int kend = min(k, kW);
  int c0 = h & ~3;
  while (c0 < kend) {
    int4 p0, p1;
    ld256cs(le + (int64_t)(c0 >> 2) * ps, p0, p1);
    const int32_t J[4] = {p0.x, p0.z, p1.x, p1.z};
    const uint32_t wb[4] = {mono_bits(__int_as_float(p0.y)), mono_bits(__int_as_float(p0.w)),
                            mono_bits(__int_as_float(p1.y)), mono_bits(__int_as_float(p1.w))};
    const float w[4] = {__int_as_float(p0.y), __int_as_float(p0.w), __int_as_float(p1.y), __int_as_float(p1.w)};
    reads += (unsigned long long)(min(c0 + 4, kend) - max(c0, h));
    uint32_t valid = 0, in = 0;
    int32_t cj[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int idx = c0 + j;
      const bool vj = idx >= h && idx < kend;
      const bool ej = w[j] <= eps;
      valid |= (uint32_t)vj << j;
      in |= (uint32_t)(vj && ej) << j;
      const bool cand = vj && ej && J[j] >= 0 && J[j] < N && J[j] != v;
      cj[j] = cand ? comp_of(comp, J[j], false, lv) : -1;
    }
    uint32_t leave = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) leave |= (uint32_t)(cj[j] >= 0 && cj[j] != cv) << j;
    int from = 0;  // first position of the chunk still to look at for ties
    if (!r.found) {
      const uint32_t stop = valid & (~in | leave);
      if (stop == 0) {  // every valid entry is dead
        h = min(c0 + 4, kend);
        c0 += 4;
        continue;
      }
      const int f = __ffs(stop) - 1;
      if (!((in >> f) & 1u)) return RowScan{false, k, kSent, kSentB, -1};  // sorted: nothing left
      int32_t Jf = 0, cf = -1;
#pragma unroll
      for (int j = 0; j < 4; ++j)  // select by an unrolled compare (a dynamic index would spill to the stack)
        if (j == f) { Jf = J[j]; cf = cj[j]; wstar = wb[j]; }
      r.found = true;
      r.h = c0 + f;
      r.best = pack_key(wstar, (uint32_t)min(v, Jf));
      r.bestb = (uint32_t)max(v, Jf);
      r.bestc = cf;
      from = f + 1;
    }
    // the tie group: valid positions >= from with the minimum's weight, up to
    // the first other weight
    uint32_t differ = 0, tie = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool vj = j >= from && ((valid >> j) & 1u);
      differ |= (uint32_t)(vj && wb[j] != wstar) << j;
      tie |= (uint32_t)(vj && wb[j] == wstar) << j;
    }
    const uint32_t before = differ ? ((1u << (__ffs(differ) - 1)) - 1u) : 0xfu;
    const uint32_t cmp = tie & leave & before;
    if (cmp) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!((cmp >> j) & 1u)) continue;
        const uint64_t kk = pack_key(wstar, (uint32_t)min(v, J[j]));
        const uint32_t bb = (uint32_t)max(v, J[j]);
        if (kk < r.best || (kk == r.best && bb < r.bestb)) { r.best = kk; r.bestb = bb; r.bestc = cj[j]; }
      }
    }
    if (differ) return r;  // the group ended inside the chunk
    c0 += 4;
  }
  if (k > kW) {
    // the candidate prefix (or the minimum's tie group) runs past the ELL
    if (!r.found) return scan_row<false, false>(nr, dr, k, eps, v, cv, max(h, kW), N, comp, 0, reads, lv);
    for (int c = kW; c < k; ++c) {  // continue the tie group of weight wstar in the graph row
      const float wc = __ldcg(dr + c);
      if (mono_bits(wc) != wstar || !(wc <= eps)) break;
      const int32_t Jc = __ldcg(nr + c);
      ++reads;
      if (Jc < 0 || Jc >= N || Jc == v) continue;
      const int32_t cc = comp_of(comp, Jc, false, lv);
      if (cc < 0 || cc == cv) continue;
      const uint64_t kk = pack_key(wstar, (uint32_t)min(v, Jc));
      const uint32_t bb = (uint32_t)max(v, Jc);
      if (kk < r.best || (kk == r.best && bb < r.bestb)) { r.best = kk; r.bestb = bb; r.bestc = cc; }
    }
  }
  if (!r.found) r.h = k;
  return r;
}

// The row kernels below take their input in ORDER: a block grabs the next
// chunk of kChunk records from a cursor, so all SMs work on neighbouring rows
// at any time and the component gathers of a cluster stay L2-resident (random
// gathers run at ~2.9e11/s while their working set is below ~64 MB, at DRAM
// rates beyond).  Outputs are staged in shared memory and written with ONE
// global reservation per chunk, so the next list keeps the order too.


// round 1 (exact mode, singletons) over the ELL; see k_offer_first
__global__ void __launch_bounds__(256) k_light_first(const int4* __restrict__ LE, int64_t ell_rows,
                                                     const int32_t* __restrict__ nbr,
                                                     const float* __restrict__ dist, int32_t ld, int32_t k, float eps,
                                                     int64_t row_begin, int64_t N, const int32_t* __restrict__ comp,
                                                     int all_core, const Rec* __restrict__ act, uint32_t n_in,
                                                     Rec* __restrict__ act_out, uint32_t* __restrict__ n_out,
                                                     uint32_t* __restrict__ grab,
                                                     uint64_t* __restrict__ Kc, uint32_t* __restrict__ Bc,
                                                     int32_t* __restrict__ tgt, unsigned long long* __restrict__ n_entries, const uint32_t* __restrict__ n_in_p = nullptr,
                                                     int chunk = kChunk, int4* __restrict__ rec1 = nullptr,
                                                     const uint32_t* __restrict__ kthL = nullptr, int skip1 = 0) {
  if (n_in_p) n_in = *n_in_p;
  __shared__ __align__(16) Rec s_rec[kChunk];
  __shared__ uint32_t s_n, s_chunk, s_base;
  unsigned long long reads = 0;
  for (;;) {
    if (threadIdx.x == 0) { s_chunk = atomicAdd(grab, 1u); s_n = 0; }
    __syncthreads();
    const uint64_t base = (uint64_t)s_chunk * chunk;
    if (base >= n_in) break;
    for (int t = 0; t < chunk; t += 256) {
      const uint64_t s = base + t + threadIdx.x;
      if (s >= n_in) continue;
      const int2 a = __ldcs(reinterpret_cast<const int2*>(act + s));
      const int32_t v = a.x;
      const int64_t i = (int64_t)v - row_begin;
      const RowScan r = scan_ell<true>(LE + ell_row(i), ell_ps(ell_rows), nbr + i * ld, dist + i * ld, k, eps, v, -1, a.y, N, comp,
                                       all_core, reads);
      if (r.found) {
        const int32_t cv = all_core ? v : gat(comp + v);
        bool skip_head = false;
        if (rec1) {  // packed record (K, B, kmin) for k_hook<true>, as the fused ELL pass writes
          const uint32_t kb = kthL[i];
          __stcg(rec1 + cv, make_int4((int)(uint32_t)r.best, (int)(uint32_t)(r.best >> 32), (int)r.bestb, (int)kb));
          // the certified minimum at the head hooks: from round 2 on it is intra
          skip_head = skip1 && r.bidx == r.h && (uint32_t)(r.best >> 32) < kb;
        } else {
          Kc[cv] = r.best;
          Bc[cv] = r.bestb;
        }
        tgt[cv] = r.bestc;
        s_rec[atomicAdd(&s_n, 1u)] = Rec{v, skip_head ? r.h + 1 : r.h};
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_n ? atomicAdd(n_out, s_n) : 0u;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < s_n; j += blockDim.x)
      __stcs(reinterpret_cast<int2*>(act_out + s_base + j), *reinterpret_cast<const int2*>(s_rec + j));
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) reads += __shfl_xor_sync(0xffffffffu, reads, o);
  if ((threadIdx.x & 31) == 0 && reads) atomicAdd(n_entries, reads);
}

// later rounds over the ELL; see k_offer_round.  CAS (one rank): the offer is
// a 128-bit CAS-minimum of (key, b) into KB[comp v] -- no offer list, no tie pass.
template <int GW, bool PIPE = false, bool CAS = false, bool LEAN = false, int GM = kGmRuntime, bool FAST = false>
__global__ void __launch_bounds__(256) k_light_round(const int4* __restrict__ LE, int64_t ell_rows,
                                                     const int32_t* __restrict__ nbr,
                                                     const float* __restrict__ dist, int32_t ld, int32_t k, float eps,
                                                     int64_t row_begin, int64_t N, const int32_t* __restrict__ comp,
                                                     const Rec* __restrict__ act, uint32_t n_in,
                                                     Rec* __restrict__ act_out, uint32_t* __restrict__ n_out,
                                                     uint32_t* __restrict__ grab, Offer* __restrict__ offers,
                                                     unsigned long long* __restrict__ Kc,
                                                     unsigned long long* __restrict__ n_entries, const uint32_t* __restrict__ n_in_p = nullptr,
                                                     int precheck = 0, ulonglong2* __restrict__ KB = nullptr,
                                                     const LocalView lv = LocalView{},
                                                     const uint8_t* __restrict__ frz = nullptr,
                                                     Rec* __restrict__ park = nullptr,
                                                     uint32_t* __restrict__ n_park = nullptr, int l2hint = 0,
                                                     int chunk = kChunk) {
  if (n_in_p) n_in = *n_in_p;
  LocalView lvh = lv;
  if (l2hint & 1) lvh.pol = l2_evict_last_policy();  // keep the component gathers' lines over the streams
  lvh.l1 = (l2hint >> 1) & 1;
  __shared__ __align__(16) Rec s_rec[kChunk];
  __shared__ __align__(16) Offer s_off[CAS ? 1 : kChunk];
  __shared__ uint32_t s_n, s_chunk, s_base;
  unsigned long long reads = 0;
  for (;;) {
    if (threadIdx.x == 0) { s_chunk = atomicAdd(grab, 1u); s_n = 0; }
    __syncthreads();
    const uint64_t base = (uint64_t)s_chunk * chunk;
    if (base >= n_in) break;
#if KDB_SLIM >= 3
#pragma unroll 1
#endif
    for (int t = 0; t < chunk; t += 256) {
      const uint64_t s = base + t + threadIdx.x;
      // CAS: the warp's offers are min-reduced over runs of lanes offering to
      // the same component before the CAS (warp-collective: every lane gets here)
      bool have = false;
      int32_t cseg = -1 - (int32_t)(threadIdx.x & 31);
      uint64_t okey = ~0ull, ob = ~0ull;
      if (s < n_in) {
      const int2 a = __ldcs(reinterpret_cast<const int2*>(act + s));
      const int32_t v = a.x;
      int32_t cv = lvh.l1 ? __ldg(comp + v) : gat(comp + v);
      if (lvh.gmap) cv = gat(lvh.gmap + cv);
      KDB_DCHECK(cv >= 0 && v >= row_begin && v < N, 8u);  // a live row is a local core vertex
      if (frz && frz[cv]) {
        // local-first phase: the component is frozen (its minimum is a remote or
        // uncertifiable edge and stays so while it only absorbs local
        // components): the row waits, head unchanged, for the global phase
        const unsigned am = __activemask();
        const int lane = threadIdx.x & 31, leader = __ffs(am) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(n_park, (uint32_t)__popc(am));
        base = __shfl_sync(am, base, leader);
        park[base + __popc(am & ((1u << lane) - 1u))] = Rec{v, a.y};
      } else {
      const int64_t i = (int64_t)v - row_begin;
      const RowScan r = (FAST && GM != kGmRuntime && GW == 4 && !PIPE)
          ? scan_ell_fast<GM>(LE + ell_row(i), ell_ps(ell_rows), nbr + i * ld, dist + i * ld, k, eps, v, cv, a.y, N,
                              comp, reads, lvh)
          : (LEAN && GW == 4 && !PIPE)
          ? scan_ell_lean(LE + ell_row(i), ell_ps(ell_rows), nbr + i * ld, dist + i * ld, k, eps, v, cv, a.y, N, comp,
                          reads, lvh)
          : scan_ell<false, GW, PIPE, GM>(LE + ell_row(i), ell_ps(ell_rows), nbr + i * ld, dist + i * ld, k, eps, v, cv, a.y,
                                                  N, comp, 0, reads, lvh);
      if (r.found) {
        const uint32_t j = atomicAdd(&s_n, 1u);
        s_rec[j] = Rec{v, r.h};
        if (CAS) {
          // (b, target component) in the second word: the CAS-minimum orders by
          // (key, b) -- equal (key, b) is the same edge, hence the same target --
          // and the hook reads the target without gathering comp[]
          have = true;
          cseg = cv;
          okey = r.best;
          ob = ((uint64_t)r.bestb << 32) | (uint32_t)r.bestc;
        } else {
          if (precheck) min_offer(Kc + cv, (unsigned long long)r.best);
          else atomicMin(Kc + cv, (unsigned long long)r.best);
          s_off[j] = Offer{cv, r.bestb, r.best};
        }
      }
      }
      }
      if (CAS) warp_min_pair128(KB, have, cseg, okey, ob);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_n ? atomicAdd(n_out, s_n) : 0u;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < s_n; j += blockDim.x) {
      __stcs(reinterpret_cast<int2*>(act_out + s_base + j), *reinterpret_cast<const int2*>(s_rec + j));
      if (!CAS) __stcs(reinterpret_cast<int4*>(offers + s_base + j), *reinterpret_cast<const int4*>(s_off + j));
    }
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) reads += __shfl_xor_sync(0xffffffffu, reads, o);
  if ((threadIdx.x & 31) == 0 && reads) atomicAdd(n_entries, reads);
}

// Later light rounds, one view, CAS offers (the single-rank default), with
// LANE REFILL: a lane whose row is finished takes the warp's next record at
// once, so every warp step scans one 4-entry chunk of some row on (nearly)
// every lane.  k_light_round runs a warp until its LONGEST row is done: ncu of
// round 3 (C4) showed 3.45 chunk steps per warp for 1.6 chunks per row, at
// 13-18 active lanes, and the chunk loop as 86% of the kernel's instructions.
// Same scan (scan_ell's entry ladder, GW = 4), same offers (the CAS-minimum of
// (key, (b, target component)) into KB[cv]) and the same next row list up to
// order; no shared memory, no block barriers: a warp grabs kRefillChunk
// records at a time from the round's cursor (records stay roughly in order,
// so the component gathers keep their L2 locality) and reserves its output
// slots with one atomic per step that finishes rows.
constexpr int kRefillChunk = 512;
#ifndef KDB_REFILL_MINB
#define KDB_REFILL_MINB 5  // blocks per SM (<= 48 registers: 40 warps, as k_light_round)
#endif
template <int GM>
__global__ void __launch_bounds__(256, KDB_REFILL_MINB) k_light_refill(const int4* __restrict__ LE, int64_t ell_rows,
                                                      const int32_t* __restrict__ nbr, const float* __restrict__ dist,
                                                      int32_t ld, int32_t k, float eps, int64_t row_begin, int64_t N,
                                                      const int32_t* __restrict__ comp, const Rec* __restrict__ act,
                                                      uint32_t n_in, Rec* __restrict__ act_out,
                                                      uint32_t* __restrict__ n_out, uint32_t* __restrict__ grab,
                                                      ulonglong2* __restrict__ KB,
                                                      unsigned long long* __restrict__ n_entries,
                                                      const uint32_t* __restrict__ n_in_p, int l2hint) {
  if (n_in_p) n_in = *n_in_p;
  LocalView lvh{};
  if (l2hint & 1) lvh.pol = l2_evict_last_policy();
  lvh.l1 = (l2hint >> 1) & 1;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int kend = min(k, kW);
  const int64_t ps = ell_ps(ell_rows);
  unsigned long long reads = 0;
  // warp queue [qpos, qend) of records (warp-uniform)
  uint32_t qpos = 0, qend = 0;
  bool exhausted = false;
  // this lane's row
  bool have = false, found = false, done = false;
  int32_t v = 0, cv = 0, bestc = -1;
  int h = 0, c0 = 0, fh = 0;
  uint32_t wstar = 0, bestb = kSentB;
  uint64_t best = kSent;
  int32_t pc = -1;  // pending offer (component, key, (b, target)) of this lane
  uint64_t pk = kSent, pb = ~0ull;
  for (;;) {
    // ---- refill: lanes without a row take the next records, in lane order
    unsigned need = __ballot_sync(0xffffffffu, !have);
    while (need && !exhausted) {
      if (qpos >= qend) {
        uint32_t c = 0;
        if (lane == 0) c = atomicAdd(grab, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        const uint64_t b0 = (uint64_t)c * kRefillChunk;
        if (b0 >= n_in) { exhausted = true; break; }
        qpos = (uint32_t)b0;
        qend = (uint32_t)(b0 + kRefillChunk < (uint64_t)n_in ? b0 + kRefillChunk : (uint64_t)n_in);
      }
      const uint32_t avail = qend - qpos;
      const uint32_t rk = __popc(need & lt);
      if (!have && rk < avail) {
        const int2 a = __ldcs(reinterpret_cast<const int2*>(act + qpos + rk));
        v = a.x;
        h = a.y;
        cv = lvh.l1 ? __ldg(comp + v) : gat(comp + v);
        KDB_DCHECK(cv >= 0 && v >= row_begin && v < N, 8u);  // a live row is a local core vertex
        c0 = h & ~3;
        found = false;
        done = false;
        best = kSent;
        bestb = kSentB;
        bestc = -1;
        fh = k;
        have = true;
      }
      qpos += min((uint32_t)__popc(need), avail);
      need = __ballot_sync(0xffffffffu, !have);
    }
    if (__ballot_sync(0xffffffffu, have) == 0) break;
    // ---- one chunk step of this lane's row (scan_ell's ladder)
    bool fin = false;
    if (have) {
      const int64_t i = (int64_t)v - row_begin;
      if (c0 < kend) {
        int4 p0, p1;
        ld256cs(LE + ell_row(i) + (int64_t)(c0 >> 2) * ps, p0, p1);
        const int32_t J[4] = {p0.x, p0.z, p1.x, p1.z};
        const float w[4] = {__int_as_float(p0.y), __int_as_float(p0.w), __int_as_float(p1.y), __int_as_float(p1.w)};
        reads += (unsigned long long)(min(c0 + 4, kend) - max(c0, h));
        int32_t cj[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int idx = c0 + j;
          const bool cand = idx >= h && idx < kend && w[j] <= eps && (uint32_t)J[j] < (uint32_t)N && J[j] != v;
          cj[j] = cand ? comp_of_m<GM>(comp, J[j], false, lvh) : -1;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int idx = c0 + j;
          if (done || idx < h || idx >= kend) continue;
          const bool leaving = cj[j] >= 0 && cj[j] != cv;
          const uint32_t wb = mono_bits(w[j]);
          if (!found) {
            if (!(w[j] <= eps)) { done = true; continue; }  // sorted: nothing left
            if (!leaving) { h = idx + 1; continue; }          // dead entry
            found = true;
            fh = idx;
            wstar = wb;
            best = pack_key(wb, (uint32_t)min(v, J[j]));
            bestb = (uint32_t)max(v, J[j]);
            bestc = cj[j];
          } else {
            if (wb != wstar) { done = true; continue; }
            if (!leaving) continue;
            const uint64_t kk = pack_key(wb, (uint32_t)min(v, J[j]));
            const uint32_t bb = (uint32_t)max(v, J[j]);
            if (kk < best || (kk == best && bb < bestb)) { best = kk; bestb = bb; bestc = cj[j]; }
          }
        }
        c0 += 4;
      }
      fin = done || c0 >= kend;
      if (fin && !done && k > kW) {
        // the candidate prefix (or the minimum's tie group) runs past the ELL (rare)
        if (!found) {
          const RowScan t = scan_row<false, false>(nbr + i * ld, dist + i * ld, k, eps, v, cv, max(h, kW), N, comp,
                                                   0, reads, lvh);
          found = t.found;
          fh = t.h;
          best = t.best;
          bestb = t.bestb;
          bestc = t.bestc;
        } else {
          const int32_t* nr = nbr + i * ld;
          const float* dr = dist + i * ld;
          for (int c = kW; c < k; ++c) {  // continue the tie group of weight wstar in the graph row
            const float wc = __ldcg(dr + c);
            if (mono_bits(wc) != wstar || !(wc <= eps)) break;
            const int32_t Jc = __ldcg(nr + c);
            ++reads;
            if (Jc < 0 || Jc >= N || Jc == v) continue;
            const int32_t cc = comp_of_m<GM>(comp, Jc, false, lvh);
            if (cc < 0 || cc == cv) continue;
            const uint64_t kk = pack_key(wstar, (uint32_t)min(v, Jc));
            const uint32_t bb = (uint32_t)max(v, Jc);
            if (kk < best || (kk == best && bb < bestb)) { best = kk; bestb = bb; bestc = cc; }
          }
        }
      }
      if (fin && found) {
        // lane-local combine: a lane's successive rows come from nearby records
        // (in later rounds mostly one component); same-address CAS loops from
        // many lanes serialise at the L2 slice, so one CAS per run of rows
        const uint64_t ob = ((uint64_t)bestb << 32) | (uint32_t)bestc;
        if (pc == cv) {
          if (best < pk || (best == pk && ob < pb)) { pk = best; pb = ob; }
        } else {
          if (pc >= 0) min_pair128(KB + pc, pk, pb);
          pc = cv;
          pk = best;
          pb = ob;
        }
      }
    }
    // ---- finished rows that found an edge stay live (head = the minimum's column)
    const unsigned out = __ballot_sync(0xffffffffu, fin && found);
    if (out) {
      uint32_t base = 0;
      const int leader = __ffs(out) - 1;
      if (lane == leader) base = atomicAdd(n_out, (uint32_t)__popc(out));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (fin && found) __stcs(reinterpret_cast<int2*>(act_out + base + __popc(out & lt)), make_int2(v, fh));
    }
    if (fin) have = false;
  }
  if (pc >= 0) min_pair128(KB + pc, pk, pb);
  for (int o = 16; o > 0; o >>= 1) reads += __shfl_xor_sync(0xffffffffu, reads, o);
  if (lane == 0 && reads) atomicAdd(n_entries, reads);
}

// Later light rounds, one view, CAS offers, QUAD PER ROW: the four lanes of a
// quad take the four entries of a chunk, so the entry ladder of scan_ell
// becomes four-lane ballots (the first valid entry that is beyond eps or
// leaving, the minimum's tie group = the valid entries of equal weight bits up
// to the first other weight) and a two-step quad minimum over (key, b).  The
// row state is quad-uniform; a warp runs 8 rows at a time, so its chunk loop
// waits for the longest of 8 rows, not of 32 (ncu of k_light_round, round 3 of
// C4: 3.45 chunk steps per warp for 1.6 per row, 13-18 active lanes, ~80
// instructions per scanned entry).  Same offers (the CAS-minimum of (key,
// (b, target component)) into KB[cv], min-reduced over runs of lanes with one
// component first) and the same next row list as k_light_round.
#ifndef KDB_QUAD_MINB
#define KDB_QUAD_MINB 5  // blocks per SM (<= 48 registers: 40 warps, as k_light_round)
#endif
template <int GM>
__global__ void __launch_bounds__(256, KDB_QUAD_MINB) k_light_quad(const int4* __restrict__ LE, int64_t ell_rows,
                                                    const int32_t* __restrict__ nbr, const float* __restrict__ dist,
                                                    int32_t ld, int32_t k, float eps, int64_t row_begin, int64_t N,
                                                    const int32_t* __restrict__ comp, const Rec* __restrict__ act,
                                                    uint32_t n_in, Rec* __restrict__ act_out,
                                                    uint32_t* __restrict__ n_out, uint32_t* __restrict__ grab,
                                                    ulonglong2* __restrict__ KB,
                                                    unsigned long long* __restrict__ n_entries,
                                                    const uint32_t* __restrict__ n_in_p, int l2hint, int chunk) {
  if (n_in_p) n_in = *n_in_p;
  LocalView lvh{};
  if (l2hint & 1) lvh.pol = l2_evict_last_policy();
  lvh.l1 = (l2hint >> 1) & 1;
  __shared__ __align__(16) Rec s_rec[kChunk];
  __shared__ uint32_t s_n, s_chunk, s_base;
  const int lane = threadIdx.x & 31, ql = lane & 3, qb = lane & ~3;
  const unsigned qmask = 0xFu << qb;
  const int kend = min(k, kW);
  const int64_t ps2 = 2 * ell_ps(ell_rows);  // chunk stride in int2 units
  const uint32_t n32 = (uint32_t)N;           // N < 2^31 (kdb_mst's check)
  unsigned long long reads = 0;
  for (;;) {
    if (threadIdx.x == 0) { s_chunk = atomicAdd(grab, 1u); s_n = 0; }
    __syncthreads();
    const uint64_t base = (uint64_t)s_chunk * chunk;
    if (base >= n_in) break;
    for (int t = 0; t < chunk; t += 64) {
      const uint64_t s = base + t + (threadIdx.x >> 2);
      bool have = false;
      int32_t cseg = -1 - lane;
      uint64_t okey = ~0ull, ob = ~0ull;
      if (s < n_in) {  // quad-uniform from here on
        const int2 a = __ldcs(reinterpret_cast<const int2*>(act + s));
        const int32_t v = a.x;
        const int h = a.y;
        const int32_t cv = lvh.l1 ? __ldg(comp + v) : gat(comp + v);
        KDB_DCHECK(cv >= 0 && v >= row_begin && v < N, 8u);  // a live row is a local core vertex
        const int64_t i = (int64_t)v - row_begin;
        const int2* le = reinterpret_cast<const int2*>(LE + ell_row(i)) + ql;
        bool found = false, done = false;
        uint32_t wstar = 0, bestb = kSentB;
        uint64_t best = kSent;
        int32_t bestc = -1;
        int fh = k;
        for (int c0 = h & ~3; c0 < kend; c0 += 4) {
          const int2 e = __ldcs(le + (int64_t)(c0 >> 2) * ps2);
          const int idx = c0 + ql;
          const int32_t J = e.x;
          const float w = __int_as_float(e.y);
          const bool valid = idx >= h && idx < kend;
          const bool in = w <= eps;
          const bool cand = valid && in && (uint32_t)J < n32 && J != v;
          const int32_t cj = cand ? comp_of_m<GM>(comp, J, false, lvh) : -1;
          const bool leave = cj >= 0 && cj != cv;
          const uint32_t wb = mono_bits(w);
          if (ql == 0) reads += (unsigned long long)(min(c0 + 4, kend) - max(c0, h));
          const unsigned bv = (__ballot_sync(qmask, valid) >> qb) & 0xFu;
          const unsigned bi = (__ballot_sync(qmask, in) >> qb) & 0xFu;
          const unsigned bl = (__ballot_sync(qmask, leave) >> qb) & 0xFu;
          int from = 0;
          if (!found) {
            const unsigned stop = bv & (~bi | bl);
            if (stop == 0) continue;  // every valid entry of the chunk is dead
            const int f = __ffs(stop) - 1;
            if (!((bi >> f) & 1u)) { done = true; break; }  // sorted: nothing left
            found = true;
            fh = c0 + f;
            wstar = __shfl_sync(qmask, wb, qb + f);
            from = f;
          }
          // the minimum's tie group in this chunk: valid positions >= from of
          // weight wstar, up to the first other weight
          const unsigned beq = (__ballot_sync(qmask, wb == wstar) >> qb) & 0xFu;
          const unsigned at = (0xFu << from) & 0xFu;
          const unsigned differ = bv & ~beq & at;
          const unsigned before = differ ? ((1u << (__ffs(differ) - 1)) - 1u) : 0xFu;
          const bool mine = ((bv & beq & bl & at & before) >> ql) & 1u;
          uint64_t kk = mine ? pack_key(wb, (uint32_t)min(v, J)) : kSent;
          uint32_t bb = mine ? (uint32_t)max(v, J) : kSentB;
          int32_t cc = cj;
#pragma unroll
          for (int o = 1; o < 4; o <<= 1) {
            const uint64_t ok = __shfl_xor_sync(qmask, kk, o);
            const uint32_t obb = __shfl_xor_sync(qmask, bb, o);
            const int32_t oc = __shfl_xor_sync(qmask, cc, o);
            if (ok < kk || (ok == kk && obb < bb)) { kk = ok; bb = obb; cc = oc; }
          }
          if (kk < best || (kk == best && bb < bestb)) { best = kk; bestb = bb; bestc = cc; }
          if (differ) { done = true; break; }
        }
        if (!done && k > kW) {
          // the candidate prefix (or the minimum's tie group) runs past the ELL
          // (rare): every lane of the quad runs the same scan
          const int32_t* nr = nbr + i * ld;
          const float* dr = dist + i * ld;
          if (!found) {
            unsigned long long tr = 0;  // entries read, counted once per quad
            const RowScan r2 = scan_row<false, false>(nr, dr, k, eps, v, cv, max(h, kW), N, comp, 0, tr, lvh);
            if (ql == 0) reads += tr;
            found = r2.found;
            fh = r2.h;
            best = r2.best;
            bestb = r2.bestb;
            bestc = r2.bestc;
          } else {
            for (int c = kW; c < k; ++c) {  // continue the tie group of weight wstar in the graph row
              const float wc = __ldcg(dr + c);
              if (mono_bits(wc) != wstar || !(wc <= eps)) break;
              const int32_t Jc = __ldcg(nr + c);
              if (ql == 0) ++reads;
              if (Jc < 0 || Jc >= N || Jc == v) continue;
              const int32_t cc2 = comp_of_m<GM>(comp, Jc, false, lvh);
              if (cc2 < 0 || cc2 == cv) continue;
              const uint64_t kk2 = pack_key(wstar, (uint32_t)min(v, Jc));
              const uint32_t bb2 = (uint32_t)max(v, Jc);
              if (kk2 < best || (kk2 == best && bb2 < bestb)) { best = kk2; bestb = bb2; bestc = cc2; }
            }
          }
        }
        if (found) {
          if (ql == 0) s_rec[atomicAdd(&s_n, 1u)] = Rec{v, fh};
          have = true;  // all four lanes: runs of lanes with one component reduce before the CAS
          cseg = cv;
          okey = best;
          ob = ((uint64_t)bestb << 32) | (uint32_t)bestc;
        }
      }
      warp_min_pair128(KB, have, cseg, okey, ob);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_n ? atomicAdd(n_out, s_n) : 0u;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < s_n; j += blockDim.x)
      __stcs(reinterpret_cast<int2*>(act_out + s_base + j), *reinterpret_cast<const int2*>(s_rec + j));
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) reads += __shfl_xor_sync(0xffffffffu, reads, o);
  if ((threadIdx.x & 31) == 0 && reads) atomicAdd(n_entries, reads);
}

// Later light rounds, one view, CAS offers, LEVEL-SYNCHRONOUS: k_light_round
// runs a warp until its longest row is done (3.45 chunk steps per warp for 1.6
// chunks per row in C4's round 3, 13-18 active lanes).  Here a block's records
// are scanned one ELL chunk per level: level 0 takes the chunk of every record's
// head; a row that found nothing there (all entries dead) is queued in shared
// memory with its component and the next chunk's column, and level L + 1 scans
// the queue of level L with full warps.  At most kW / 4 levels.  Queue pushes
// keep the warp's lane order (ballot + one shared atomic per warp), so runs of
// one component stay adjacent for warp_min_pair128.  Same scan, offers and next
// row list (up to order) as k_light_round<4, false, true>.
#ifndef KDB_LVL_MINB
#define KDB_LVL_MINB 5
#endif
template <int GM>
__global__ void __launch_bounds__(256, KDB_LVL_MINB) k_light_lvl(const int4* __restrict__ LE, int64_t ell_rows,
                                                   const int32_t* __restrict__ nbr, const float* __restrict__ dist,
                                                   int32_t ld, int32_t k, float eps, int64_t row_begin, int64_t N,
                                                   const int32_t* __restrict__ comp, const Rec* __restrict__ act,
                                                   uint32_t n_in, Rec* __restrict__ act_out,
                                                   uint32_t* __restrict__ n_out, uint32_t* __restrict__ grab,
                                                   ulonglong2* __restrict__ KB,
                                                   unsigned long long* __restrict__ n_entries,
                                                   const uint32_t* __restrict__ n_in_p, int l2hint, int chunk) {
  if (n_in_p) n_in = *n_in_p;
  LocalView lvh{};
  if (l2hint & 1) lvh.pol = l2_evict_last_policy();
  lvh.l1 = (l2hint >> 1) & 1;
  constexpr int kLevels = kW / 4 + 1;
  __shared__ __align__(16) Rec s_rec[kChunk];
  __shared__ __align__(8) int2 s_qa[2][kChunk];  // (v, next column)
  __shared__ int32_t s_qc[2][kChunk];            // comp[v]
  __shared__ uint32_t s_n, s_chunk, s_base, s_nq[kLevels];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long reads = 0;
  for (;;) {
    if (threadIdx.x == 0) { s_chunk = atomicAdd(grab, 1u); s_n = 0; }
    if (threadIdx.x < kLevels) s_nq[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)s_chunk * chunk;
    if (base >= n_in) break;
    uint32_t n_items = (uint32_t)min((uint64_t)chunk, (uint64_t)n_in - base);
    for (int level = 0; n_items; ++level) {
      const int q = level & 1;
      for (uint32_t t = 0; t < n_items; t += 256) {
        const uint32_t s = t + threadIdx.x;
        bool have = false, cont = false;
        int32_t cseg = -1 - lane, v = 0, cv = 0;
        int rh = 0;
        uint64_t okey = ~0ull, ob = ~0ull;
        if (s < n_items) {
          int hh;
          if (level == 0) {
            const int2 a = __ldcs(reinterpret_cast<const int2*>(act + base + s));
            v = a.x;
            hh = a.y;
            cv = lvh.l1 ? __ldg(comp + v) : gat(comp + v);
          } else {
            const int2 a = s_qa[q ^ 1][s];
            v = a.x;
            hh = a.y;
            cv = s_qc[q ^ 1][s];
          }
          KDB_DCHECK(cv >= 0 && v >= row_begin && v < N, 8u);
          const int64_t i = (int64_t)v - row_begin;
          const RowScan r = scan_ell<false, 4, false, GM, true>(LE + ell_row(i), ell_ps(ell_rows), nbr + i * ld,
                                                                dist + i * ld, k, eps, v, cv, hh, N, comp, 0, reads, lvh);
          rh = r.h;
          if (r.cont) cont = true;
          else if (r.found) {
            have = true;
            cseg = cv;
            okey = r.best;
            ob = ((uint64_t)r.bestb << 32) | (uint32_t)r.bestc;
          }
        }
        const unsigned mc = __ballot_sync(0xffffffffu, cont);
        if (mc && level + 1 < kLevels) {
          uint32_t b = 0;
          if (lane == 0) b = atomicAdd(&s_nq[level], (uint32_t)__popc(mc));
          b = __shfl_sync(0xffffffffu, b, 0);
          if (cont) {
            const uint32_t j = b + __popc(mc & lt);
            s_qa[q][j] = make_int2(v, rh);
            s_qc[q][j] = cv;
          }
        }
        const unsigned mf = __ballot_sync(0xffffffffu, have);
        if (mf) {
          uint32_t b = 0;
          if (lane == 0) b = atomicAdd(&s_n, (uint32_t)__popc(mf));
          b = __shfl_sync(0xffffffffu, b, 0);
          if (have) s_rec[b + __popc(mf & lt)] = Rec{v, rh};
        }
        warp_min_pair128(KB, have, cseg, okey, ob);
      }
      __syncthreads();
      n_items = level + 1 < kLevels ? s_nq[level] : 0u;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_n ? atomicAdd(n_out, s_n) : 0u;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < s_n; j += blockDim.x)
      __stcs(reinterpret_cast<int2*>(act_out + s_base + j), *reinterpret_cast<const int2*>(s_rec + j));
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) reads += __shfl_xor_sync(0xffffffffu, reads, o);
  if ((threadIdx.x & 31) == 0 && reads) atomicAdd(n_entries, reads);
}

// k_light_lvl with a POOL instead of levels: every block step scans one ELL
// chunk of up to `chunk` rows -- the rows the previous step left unfinished
// (kept in shared memory with their component and next column) plus as many
// new records from the round's cursor as fill the step.  Deep levels then run
// with full warps too (k_light_lvl's level 2 / 3 keep 5 / 2 of a block's 8
// warps busy).  `grab` counts RECORDS here, not chunks.
template <int GM, bool FAST = false>
__global__ void __launch_bounds__(256, KDB_LVL_MINB) k_light_pool(const int4* __restrict__ LE, int64_t ell_rows,
                                                    const int32_t* __restrict__ nbr, const float* __restrict__ dist,
                                                    int32_t ld, int32_t k, float eps, int64_t row_begin, int64_t N,
                                                    const int32_t* __restrict__ comp, const Rec* __restrict__ act,
                                                    uint32_t n_in, Rec* __restrict__ act_out,
                                                    uint32_t* __restrict__ n_out, uint32_t* __restrict__ grab,
                                                    ulonglong2* __restrict__ KB,
                                                    unsigned long long* __restrict__ n_entries,
                                                    const uint32_t* __restrict__ n_in_p, int l2hint, int chunk) {
  if (n_in_p) n_in = *n_in_p;
  LocalView lvh{};
  if (l2hint & 1) lvh.pol = l2_evict_last_policy();
  lvh.l1 = (l2hint >> 1) & 1;
  __shared__ __align__(16) Rec s_rec[kChunk];
  __shared__ __align__(8) int2 s_qa[2][kChunk];  // (v, next column)
  __shared__ int32_t s_qc[2][kChunk];            // comp[v]
  __shared__ uint32_t s_n, s_in, s_base, s_np[2];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long reads = 0;
  if (threadIdx.x < 2) s_np[threadIdx.x] = 0;
  __syncthreads();
  bool dry = false;  // the cursor ran past the list (block-uniform)
  for (int p = 0;; p ^= 1) {
    const uint32_t np = s_np[p];
    const uint32_t want = dry ? 0u : (uint32_t)chunk - np;
    if (threadIdx.x == 0) {
      s_in = want ? atomicAdd(grab, want) : n_in;
      s_n = 0;
      s_np[p ^ 1] = 0;
    }
    __syncthreads();
    const uint32_t b = s_in;
    const uint32_t avail = b < n_in ? min(want, n_in - b) : 0u;
    if (avail < want || !want) dry = true;
    const uint32_t n_items = np + avail;
    if (n_items == 0) break;
    for (uint32_t t = 0; t < n_items; t += 256) {
      const uint32_t s = t + threadIdx.x;
      bool have = false, cont = false;
      int32_t cseg = -1 - lane, v = 0, cv = 0;
      int rh = 0;
      uint64_t okey = ~0ull, ob = ~0ull;
      if (s < n_items) {
        int hh;
        if (s >= np) {
          const int2 a = __ldcs(reinterpret_cast<const int2*>(act + b + (s - np)));
          v = a.x;
          hh = a.y;
          cv = lvh.l1 ? __ldg(comp + v) : gat(comp + v);
        } else {
          const int2 a = s_qa[p][s];
          v = a.x;
          hh = a.y;
          cv = s_qc[p][s];
        }
        KDB_DCHECK(cv >= 0 && v >= row_begin && v < N, 8u);
        const int64_t i = (int64_t)v - row_begin;
        const RowScan r = FAST
            ? scan_ell_fast<GM, true>(LE + ell_row(i), ell_ps(ell_rows), nbr + i * ld, dist + i * ld, k, eps, v, cv, hh, N,
                                      comp, reads, lvh)
            : scan_ell<false, 4, false, GM, true>(LE + ell_row(i), ell_ps(ell_rows), nbr + i * ld, dist + i * ld, k, eps,
                                                  v, cv, hh, N, comp, 0, reads, lvh);
        rh = r.h;
        if (r.cont) cont = true;
        else if (r.found) {
          have = true;
          cseg = cv;
          okey = r.best;
          ob = ((uint64_t)r.bestb << 32) | (uint32_t)r.bestc;
        }
      }
      const unsigned mc = __ballot_sync(0xffffffffu, cont);
      if (mc) {
        uint32_t bq = 0;
        if (lane == 0) bq = atomicAdd(&s_np[p ^ 1], (uint32_t)__popc(mc));
        bq = __shfl_sync(0xffffffffu, bq, 0);
        if (cont) {
          const uint32_t j = bq + __popc(mc & lt);
          s_qa[p ^ 1][j] = make_int2(v, rh);
          s_qc[p ^ 1][j] = cv;
        }
      }
      const unsigned mf = __ballot_sync(0xffffffffu, have);
      if (mf) {
        uint32_t bf = 0;
        if (lane == 0) bf = atomicAdd(&s_n, (uint32_t)__popc(mf));
        bf = __shfl_sync(0xffffffffu, bf, 0);
        if (have) s_rec[bf + __popc(mf & lt)] = Rec{v, rh};
      }
      warp_min_pair128(KB, have, cseg, okey, ob);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_n ? atomicAdd(n_out, s_n) : 0u;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < s_n; j += blockDim.x)
      __stcs(reinterpret_cast<int2*>(act_out + s_base + j), *reinterpret_cast<const int2*>(s_rec + j));
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) reads += __shfl_xor_sync(0xffffffffu, reads, o);
  if ((threadIdx.x & 31) == 0 && reads) atomicAdd(n_entries, reads);
}

// in-edge lists: scan the live in-entries of target t, drop intra entries
// (swap-remove; they never revive), offer the minimum leaving one.
__global__ void k_offer_in(const unsigned long long* __restrict__ in_off, int32_t* __restrict__ in_len,
                           int32_t* __restrict__ in_src, float* __restrict__ in_w,
                           const int32_t* __restrict__ comp, const int32_t* __restrict__ act_in,
                           uint32_t n_in, int32_t* __restrict__ act_out, uint32_t* __restrict__ n_out,
                           Offer* __restrict__ offers, uint32_t* __restrict__ n_off,
                           unsigned long long* __restrict__ Kc, const uint32_t* __restrict__ n_in_p = nullptr) {
  if (n_in_p) n_in = *n_in_p;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n_in; base += gridDim.x * blockDim.x) {
    const uint32_t s = base + threadIdx.x;
    bool found = false, keep = false;
    uint64_t best = kSent;
    uint32_t bestb = kSentB;
    int32_t t = -1, ct = -1;
    if (s < n_in) {
      t = act_in[s];
      ct = comp[t];
      const unsigned long long o = in_off[t];
      int32_t len = in_len[t];
      int32_t e = 0;
      while (e < len) {
        const int32_t u = in_src[o + e];
        if (comp[u] == ct) {  // intra for good: swap-remove
          --len;
          in_src[o + e] = in_src[o + len];
          in_w[o + e] = in_w[o + len];
          continue;
        }
        const uint64_t kk = pack_key(mono_bits(in_w[o + e]), (uint32_t)min(u, t));
        const uint32_t bb = (uint32_t)max(u, t);
        if (kk < best || (kk == best && bb < bestb)) { best = kk; bestb = bb; }
        found = true;
        ++e;
      }
      in_len[t] = len;
      keep = len > 0;
    }
    const uint32_t a = block_reserve(n_out, keep);
    if (keep) act_out[a] = t;
    const uint32_t o2 = block_reserve(n_off, found);
    if (found) {
      offers[o2] = Offer{ct, bestb, best};
      atomicMin(Kc + ct, (unsigned long long)best);
    }
  }
}

// ============================================================================
// a4: tie pass (b of the minimum key); the offer count is read on the device
// ============================================================================
__global__ void k_tie(const Offer* __restrict__ offers, const uint32_t* __restrict__ n_p,
                      const uint64_t* __restrict__ Kc, uint32_t* __restrict__ Bc) {
  const uint32_t n = *n_p;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const Offer o = offers[s];
    if (o.key == gat(Kc + o.c)) atomicMin(Bc + o.c, o.b);
  }
}

// stall fallback (exact mode): offer EVERY live leaving entry of the active
// rows to both endpoint components (rows outside the active list have none)
__global__ void k_sweep(const int32_t* __restrict__ nbr, const float* __restrict__ dist, int32_t ld, int32_t k, float eps,
                        int64_t row_begin, int64_t N, const int32_t* __restrict__ comp,
                        const Rec* __restrict__ act, uint32_t n_act, unsigned long long* __restrict__ Kc,
                        uint32_t* __restrict__ Bc, int tie_phase) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_act; s += gridDim.x * blockDim.x) {
    const int64_t v = act[s].v;
    const int64_t i = v - row_begin;
    const int32_t cv = comp[v];
    for (int32_t c = act[s].h; c < k; ++c) {
      const float w = __ldg(dist + i * ld + c);
      if (!(w <= eps)) break;
      const int64_t J = __ldg(nbr + i * ld + c);
      if (J < 0 || J >= N || J == v) continue;
      const int32_t cj = comp[J];
      if (cj < 0 || cj == cv) continue;
      const uint64_t kk = pack_key(mono_bits(w), (uint32_t)min(v, J));
      const uint32_t bb = (uint32_t)max(v, J);
      if (!tie_phase) {
        atomicMin(Kc + cv, (unsigned long long)kk);
        atomicMin(Kc + cj, (unsigned long long)kk);
      } else {
        if (kk == Kc[cv]) atomicMin(Bc + cv, bb);
        if (kk == Kc[cj]) atomicMin(Bc + cj, bb);
      }
    }
  }
}

// ============================================================================
// sim backend: elementwise MIN of per-virtual-rank partials
// ============================================================================

__global__ void k_min_into_u64(uint64_t* __restrict__ d, const uint64_t* __restrict__ s, int64_t n,
                               const int64_t* __restrict__ np = nullptr) {
  if (np) n = *np;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    if (s[c] < d[c]) d[c] = s[c];
}
__global__ void k_min_into_u32(uint32_t* __restrict__ d, const uint32_t* __restrict__ s, int64_t n,
                               const int64_t* __restrict__ np = nullptr) {
  if (np) n = *np;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    if (s[c] < d[c]) d[c] = s[c];
}

// ============================================================================
// a5: hook (break symmetry) + MSF emission
// ============================================================================


__device__ __forceinline__ bool certified(uint64_t K, const uint32_t* kmin, int64_t c) {
  return kmin == nullptr || (uint32_t)(K >> 32) < gat(kmin + c);
}

// tgt != null: the hook target of every offering component is known (round 1,
// written by its single offer), so t = tgt[c] and "mutual" is tgt[t] == c.
// Otherwise t is found from the selected edge's endpoints.
// Components are taken in chunks of kHookChunk; a chunk's emitted MSF edges are
// staged in shared memory and written with one reservation; the round counters
// are summed in registers and flushed once per warp at the end.
constexpr int kHookChunk = 1024;

template <bool PACKED>
__global__ void __launch_bounds__(256) k_hook(int64_t C, const uint64_t* __restrict__ Kc, const uint32_t* __restrict__ Bc,
                       const int32_t* __restrict__ tgt, const uint32_t* __restrict__ kmin /* null = all certified */,
                       const int32_t* __restrict__ comp, int32_t* __restrict__ parent,
                       uint64_t* __restrict__ e_key, float* __restrict__ e_w, int64_t e_cap,
                       RoundCounters* __restrict__ ctr, const int64_t* __restrict__ Cp,
                       const int4* __restrict__ rec1, const ulonglong2* __restrict__ KB = nullptr,
                       uint8_t* __restrict__ frz = nullptr, int hchunk = kHookChunk,
                       const int32_t* __restrict__ gmap = nullptr) {
  if (Cp) C = *Cp;
  __shared__ uint64_t s_key[kHookChunk];
  __shared__ uint32_t s_w[kHookChunk];
  __shared__ uint32_t s_n, s_base;
  uint32_t n_off = 0, n_unc = 0, n_hook = 0;
#ifdef KDB_INJECT_OVERRUN
  // guard self-test build only (tools/guard_selftest.sh): one write past e_key
  if (blockIdx.x == 0 && threadIdx.x == 0) e_key[e_cap + 32] = 0ull;  // e_key holds e_cap + 1: this is in the guard
#endif
  for (int64_t chunk = blockIdx.x; chunk * hchunk < C; chunk += gridDim.x) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int t = 0; t < hchunk; t += blockDim.x) {
      const int64_t c = chunk * hchunk + t + threadIdx.x;
      if (c >= C) continue;
      uint64_t K;
      uint32_t Bown = 0, kbown = kInfBits;
      int32_t tKB = -1;
      if (PACKED) {  // round 1, single rank: (K, B, kmin) of a component in one 16-B record
        const int4 q = __ldcs(rec1 + c);
        K = (uint64_t)(uint32_t)q.x | ((uint64_t)(uint32_t)q.y << 32);
        Bown = (uint32_t)q.z;
        kbown = (uint32_t)q.w;
      } else if (KB) {  // one rank, CAS offers: (key, b << 32 | target) of a component in one 16-B word
        const ulonglong2 q = KB[c];
        K = q.x;
        Bown = (uint32_t)(q.y >> 32);
        tKB = (int32_t)(uint32_t)q.y;
      } else {
        K = Kc[c];
      }
      int32_t p = (int32_t)c;
      if (K != kSent) {
        ++n_off;
        if (PACKED ? !((uint32_t)(K >> 32) < kbown) : !certified(K, kmin, c)) {
          ++n_unc;
          // local-first phase: an uncertified component waits for the global
          // phase (its true minimum may be an in-edge from another rank's row)
          if (frz) frz[c] = 1;
        } else if (frz && (PACKED || KB ? (PACKED ? tgt[c] : tKB) : kRemote) == kRemote) {
          // local-first phase: the minimum leaves the rank -- frozen (a frozen
          // component never hooks, so it stays a root and keeps that minimum
          // while local components hook into it)
          ++n_unc;
          frz[c] = 1;
        } else {
          const uint32_t a = (uint32_t)K;
          const uint32_t b = (PACKED || KB) ? Bown : Bc[c];
          int32_t t2;
          if (tgt) {
            t2 = tgt[c];
          } else if (KB) {
            t2 = tKB;
          } else {
            auto cur = [&](uint32_t y) {  // current component of vertex y
              const int32_t q = gat(comp + y);
              return gmap ? gat(gmap + q) : q;
            };
            const int32_t x = (cur(a) == (int32_t)c) ? (int32_t)b : (int32_t)a;
            t2 = cur((uint32_t)x);
          }
          KDB_DCHECK(t2 >= 0 && t2 < C, 1u);
          bool mutual, cert_t = true;
          if (PACKED) {  // one random 16-B read of the target's record
            const int4 q = __ldcg(rec1 + t2);
            const uint64_t Kt = (uint64_t)(uint32_t)q.x | ((uint64_t)(uint32_t)q.y << 32);
            const uint32_t Bt = (uint32_t)q.z;
            cert_t = Kt != kSent && (uint32_t)(Kt >> 32) < (uint32_t)q.w;
            if (cert_t && (Kt > K || (Kt == K && Bt > b))) ctr->violation = 1u;
            mutual = cert_t && Kt == K && Bt == b;
          } else if (KB) {  // exact mode (CAS offers imply it): as below, one 16-B read of t
            const ulonglong2 q = __ldcg(KB + t2);
            const uint64_t Kt = q.x;
            cert_t = Kt != kSent && certified(Kt, kmin, t2);
            const uint32_t Bt = (uint32_t)(q.y >> 32);
            if (cert_t && (Kt > K || (Kt == K && Bt > b))) ctr->violation = 1u;
            mutual = cert_t && Kt == K && Bt == b;
          } else if (kmin) {  // exact mode: t may abstain; also audit the promise
            const uint64_t Kt = gat(Kc + t2);
            cert_t = Kt != kSent && certified(Kt, kmin, t2);
            // t's true minimum is <= the edge c selected (that edge is incident
            // to t); a larger key means t's offer missed an incident edge --
            // impossible under a true EXACT promise, and the only way a hook
            // cycle longer than a mutual pair could form (Fig. cycle).
            const uint32_t Bt = cert_t ? gat(Bc + t2) : 0u;
            if (cert_t && (Kt > K || (Kt == K && Bt > b))) ctr->violation = 1u;
            mutual = cert_t && Kt == K && Bt == b;
          } else if (tgt) {
            mutual = gat(tgt + t2) == (int32_t)c;
          } else {
            mutual = gat(Kc + t2) == K && gat(Bc + t2) == b;
          }
          if (!(mutual && c < t2)) {
            p = t2;
            ++n_hook;
            const uint32_t j = atomicAdd(&s_n, 1u);
            s_key[j] = ((uint64_t)b << 32) | (uint32_t)(K >> 32);  // (b, w bits): the sort payload
            s_w[j] = a;                                               // a: the sort key
          }
        }
      }
      parent[c] = p;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_n ? atomicAdd(&ctr->msf_count, s_n) : 0u;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < s_n; j += blockDim.x) {
      if ((int64_t)(s_base + j) < e_cap) {
        e_key[s_base + j] = s_key[j];
        reinterpret_cast<uint32_t*>(e_w)[s_base + j] = s_w[j];
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    n_off += __shfl_xor_sync(0xffffffffu, n_off, o);
    n_unc += __shfl_xor_sync(0xffffffffu, n_unc, o);
    n_hook += __shfl_xor_sync(0xffffffffu, n_hook, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (n_off) atomicAdd(&ctr->offered, n_off);
    if (n_unc) atomicAdd(&ctr->uncertified, n_unc);
    if (n_hook) atomicAdd(&ctr->hooks, n_hook);
  }
}

// ============================================================================
// a6: pointer jumping, dense renumbering, relabel
// ============================================================================
// Path halving on the hook forest.  Concurrent writes only ever replace a
// parent pointer by one of its ancestors, so every thread still reaches the
// same root; stale reads are ancestors too, so the loop terminates.  The root
// goes to a SEPARATE array: another thread's halving write may land on
// parent[c] after c found its root, so parent[c] itself is not final.
__global__ void k_jump(int64_t C, int32_t* parent, int32_t* __restrict__ rootof, RoundCounters* ctr,
                       const int64_t* __restrict__ Cp = nullptr, int32_t* __restrict__ flag = nullptr) {
  // flag != null (dense renumbering): also the root flags the scan needs, over
  // the host bound C with zeros beyond the true count (was k_root_flags)
  const int64_t Cb = C;
  if (Cp) C = *Cp;
  if (flag)
    for (int64_t c = C + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < Cb; c += (int64_t)gridDim.x * blockDim.x)
      flag[c] = 0;
  volatile int32_t* P = parent;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    int32_t x = (int32_t)c;
    int64_t steps = 0;
    while (true) {
      const int32_t p = P[x];
      if (p == x) break;
      const int32_t gp = P[p];
      if (gp == p) { x = p; break; }
      P[x] = gp;
      x = gp;
      if (++steps > C) {  // defence in depth: never spin on a cycle
        ctr->violation = 2u;
        break;
      }
    }
    KDB_DCHECK(x >= 0 && x < C, 4u);
    rootof[c] = x;
    if (flag) flag[c] = (x == (int32_t)c);
  }
}


// new per-component arrays: cmin/kmin are minima over the merged tree
__global__ void k_merge(int64_t C, const int32_t* __restrict__ rootof, const int32_t* __restrict__ newid,
                        const int32_t* __restrict__ cmin, const uint32_t* __restrict__ kmin,
                        int32_t* __restrict__ cmin2, uint32_t* __restrict__ kmin2, int32_t* __restrict__ map, const int64_t* __restrict__ Cp = nullptr,
                        const uint8_t* __restrict__ frz = nullptr, uint8_t* __restrict__ frz2 = nullptr) {
  if (Cp) C = *Cp;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    KDB_DCHECK(rootof[c] >= 0 && rootof[c] < C, 2u);
    const int32_t r = newid ? gat(newid + rootof[c]) : rootof[c];  // sparse ids: the root itself
    KDB_DCHECK(r >= 0 && r < C, 2u);
    map[c] = r;
    atomicMin(cmin2 + r, cmin[c]);
    if (kmin) {
      const uint32_t km = kmin[c];
      if (km != kInfBits) atomicMin(kmin2 + r, km);  // kmin2 starts at +inf
    }
    if (frz && frz[c]) frz2[r] = 1;  // frozen components are roots; the flag stays with them
  }
}

// number of core vertices below each position pos[i] (a rank's first global
// dense id): woff[p >> 5] + the core bits below p in its word
__global__ void k_core_below(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ woff,
                             const int64_t* __restrict__ pos, int n, int64_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t p = pos[i];
  const uint32_t b = (p & 31) ? __popc(bits[p >> 5] & ((1u << (p & 31)) - 1u)) : 0u;
  out[i] = (int64_t)woff[p >> 5] + b;
}

// MSF edges (e_w = a, e_key = b << 32 | w bits) whose smaller endpoint a lies
// in [lo, hi), compacted (multi-rank output: each rank returns its a-range)
__global__ void k_keep_a_range(const uint64_t* __restrict__ e_key, const uint32_t* __restrict__ e_a, int64_t n,
                               int64_t lo, int64_t hi, uint64_t* __restrict__ o_key, uint32_t* __restrict__ o_a,
                               uint32_t* __restrict__ cnt) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool keep = false;
    uint32_t a = 0;
    if (i < n) {
      a = e_a[i];
      keep = (int64_t)a >= lo && (int64_t)a < hi;
    }
    const uint32_t slot = block_reserve(cnt, keep);
    if (keep) {
      o_key[slot] = e_key[i];
      o_a[slot] = a;
    }
  }
}

// The contraction's bookkeeping in one launch (was k_count_roots + two fills +
// the offer-slot fill + a memset): the new component count -- from the root
// scan (dense ids) or unchanged (sparse) -- and the next round's
// per-component slots: cmin2 / kmin2 (minima over the merged trees; before
// k_merge), the offer slots (Kc/Bc, or the CAS words KB) and the frozen flags.
__global__ void k_round_fill(int64_t C_bound, const int64_t* __restrict__ Cd, const int32_t* __restrict__ newid,
                             const int32_t* __restrict__ flag, int64_t* __restrict__ Cn_out, int32_t* __restrict__ cmin2,
                             uint32_t* __restrict__ kmin2, uint64_t* __restrict__ Kc, uint32_t* __restrict__ Bc,
                             ulonglong2* __restrict__ KB, uint8_t* __restrict__ frz2) {
  const int64_t Cc = *Cd;
  const int64_t Cn = newid ? (Cc > 0 ? (int64_t)newid[Cc - 1] + flag[Cc - 1] : 0) : Cc;
  if (blockIdx.x == 0 && threadIdx.x == 0) *Cn_out = Cn;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C_bound; c += (int64_t)gridDim.x * blockDim.x) {
    if (frz2) frz2[c] = 0;
    if (c >= Cn) continue;
    cmin2[c] = INT32_MAX;
    if (kmin2) kmin2[c] = kInfBits;
    if (KB) {
      KB[c] = make_ulonglong2(kSent, ~0ull);
    } else {
      Kc[c] = kSent;
      Bc[c] = kSentB;
    }
  }
}

// start of a row round: the rank's output counters; with g, the round's hook counters
__global__ void k_round_reset(RoundCounters* __restrict__ rc, int cur, RoundCounters* __restrict__ g) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  rc->na[cur ^ 1] = 0;
  rc->ni[cur ^ 1] = 0;
  rc->n_off = 0;
  rc->grab = 0;
  if (g) g->hooks = g->offered = g->uncertified = g->n_roots = 0;
}

// comp[v] += delta for the core vertices of a row range (local <-> global ids)
__global__ void k_shift_comp(int32_t* __restrict__ comp, int64_t n, int32_t delta) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = comp[v];
    if (c >= 0) comp[v] = c + delta;
  }
}

__global__ void k_fill_i32(int32_t* __restrict__ p, int64_t n, int32_t val, const int64_t* __restrict__ np = nullptr) {
  if (np) n = *np;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x)
    p[c] = val;
}

// comp[v] = m2[m1[comp[v]]] (m2 optional) for every comp[v] >= 0.  Each thread
// takes 8 consecutive vertices per step (two int4 loads, 8 independent
// gathers in flight): the loop is bound by gather latency otherwise.
__global__ void k_relabel(int64_t N, int32_t* __restrict__ comp, const int32_t* __restrict__ m1,
                          const int32_t* __restrict__ m2) {
  const int64_t n8 = ((uintptr_t)comp & 15u) ? 0 : N / 8;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n8; q += (int64_t)gridDim.x * blockDim.x) {
    int4* p = reinterpret_cast<int4*>(comp) + 2 * q;
    int4 a = p[0], b = p[1];
    int32_t c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    // read-only maps through L1 (__ldg): when few components remain, 64M
    // gathers hit a handful of lines, which would serialise on their L2 slices
    const int32_t c0[8] = {c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]};
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = c[j] >= 0 ? __ldg(m1 + c[j]) : c[j];
    if (m2) {
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = c[j] >= 0 ? __ldg(m2 + c[j]) : c[j];
    }
    // sparse ids (late rounds): most vertices keep theirs -- store only changes
    bool ch0 = false, ch1 = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) { ch0 |= c[j] != c0[j]; ch1 |= c[j + 4] != c0[j + 4]; }
    if (ch0) p[0] = make_int4(c[0], c[1], c[2], c[3]);
    if (ch1) p[1] = make_int4(c[4], c[5], c[6], c[7]);
  }
  for (int64_t v = n8 * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N;
       v += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = comp[v];
    if (c >= 0) {
      c = __ldg(m1 + c);
      if (m2) c = __ldg(m2 + c);
      comp[v] = c;
    }
  }
}

// ============================================================================
// a9 / a11: canonical labels, MSF output, exact weight
// ============================================================================

// MSF output in (a, b) order: radix sort on the 32-bit a (only ceil(log2 N)
// bits) carrying (b, w) as a 64-bit payload, then each run of equal a (tiny:
// a vertex is the smaller endpoint of few MSF edges) is sorted by b in place.
// ka = the sorted a (the caller's mst_a); splits the (b, w) payload into mst_b /
// mst_w and sorts every run of equal a by b
constexpr int kRunMax = 32;  // longer runs of equal a go to the segmented sort
// Every thread's work is bounded by kRunMax + log2(m), whatever the run lengths
// (a hub vertex can be the smaller endpoint of millions of MSF edges):
//   * a run start i scans at most kRunMax + 1 entries forward; a short run
//     [i, j) is insertion-sorted by b; a long run's end comes from a binary
//     search (ka is sorted), the run is recorded as a segment and the start
//     thread unpacks only its first kRunMax + 1 entries;
//   * any other entry scans at most kRunMax entries back: if that reaches its
//     run start, the start thread owns it; otherwise it belongs to a long run
//     and unpacks itself.
// a11 (dense forests): counting sort of the emitted edges by their smaller
// endpoint a -- each edge's rank inside its bucket from the atomic it counts
// with, then a scatter through the scanned counts; the unpack below sorts each
// run of equal a by b, so the atomic order never reaches the output
__global__ void k_msf_count(int64_t m, const uint32_t* __restrict__ a, uint32_t* __restrict__ cnt,
                            uint32_t* __restrict__ pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    pos[i] = atomicAdd(cnt + a[i], 1u);
}
__global__ void k_msf_scatter(int64_t m, const uint32_t* __restrict__ a, const unsigned long long* __restrict__ vb,
                              const uint32_t* __restrict__ off, const uint32_t* __restrict__ pos,
                              uint32_t* __restrict__ ka, unsigned long long* __restrict__ vb2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t ai = a[i];
    const uint32_t d = off[ai] + pos[i];
    ka[d] = ai;
    vb2[d] = vb[i];
  }
}

__global__ void k_msf_unpack(int64_t m, const uint32_t* __restrict__ ka, const unsigned long long* __restrict__ vb,
                             uint32_t* __restrict__ b, float* __restrict__ w, int32_t* __restrict__ seg_b,
                             int32_t* __restrict__ seg_e, uint32_t* __restrict__ nseg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t ai = ka[i];
    if (i > 0 && ka[i - 1] == ai) {  // not a run start
      int64_t q = i - 1;
      while (q > 0 && i - q <= kRunMax && ka[q - 1] == ai) --q;
      if (i - q <= kRunMax) continue;  // within kRunMax of the start: the start thread's entry
      const unsigned long long x = vb[i];  // deep inside a long run: unpack in place
      b[i] = (uint32_t)(x >> 32);
      w[i] = __uint_as_float((uint32_t)x);
      continue;
    }
    int64_t j = i + 1;
    while (j < m && j - i <= kRunMax && ka[j] == ai) ++j;
    if (j - i > kRunMax) {  // a hub: its end by binary search over the sorted keys
      int64_t lo = j, hi = m;  // first index in [j, m) with ka > ai
      while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (ka[mid] > ai) hi = mid; else lo = mid + 1;
      }
      for (int64_t p = i; p <= i + kRunMax; ++p) {  // the head; the rest unpacks itself
        const unsigned long long x = vb[p];
        b[p] = (uint32_t)(x >> 32);
        w[p] = __uint_as_float((uint32_t)x);
      }
      const uint32_t s = atomicAdd(nseg, 1u);
      seg_b[s] = (int32_t)i;
      seg_e[s] = (int32_t)lo;
      continue;
    }
    for (int64_t p = i; p < j; ++p) {  // insertion sort of the run [i, j) by b
      const unsigned long long x = vb[p];
      int64_t q = p;
      while (q > i && (uint32_t)(b[q - 1]) > (uint32_t)(x >> 32)) {
        b[q] = b[q - 1];
        w[q] = w[q - 1];
        --q;
      }
      b[q] = (uint32_t)(x >> 32);
      w[q] = __uint_as_float((uint32_t)x);
    }
  }
}

// the sorted long runs back into the output (one block per run)
__global__ void k_copy_segments(const int32_t* __restrict__ seg_b, const int32_t* __restrict__ seg_e, uint32_t nseg,
                                const uint32_t* __restrict__ kout, const float* __restrict__ vout,
                                uint32_t* __restrict__ b, float* __restrict__ w) {
  for (uint32_t s = blockIdx.x; s < nseg; s += gridDim.x)
    for (int32_t p = seg_b[s] + threadIdx.x; p < seg_e[s]; p += blockDim.x) {
      b[p] = kout[p];
      w[p] = vout[p];
    }
}

// exact sum: integer mantissas bucketed by biased exponent (order independent)
__global__ void k_wbuckets(int64_t m, const float* __restrict__ w, unsigned long long* __restrict__ bk) {
  __shared__ unsigned long long sb[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) sb[t] = 0;
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = __float_as_uint(w[e]) & 0x7fffffffu;
    const uint32_t ex = u >> 23;
    uint32_t man = u & 0x7fffffu;
    if (ex) man |= 0x800000u;
    // lanes sharing an exponent pre-sum (32 x 2^24 < 2^32) -> one smem atomic each
    const unsigned grp = __match_any_sync(__activemask(), ex);
    const uint32_t sum = __reduce_add_sync(grp, man);
    if ((threadIdx.x & 31) == __ffs(grp) - 1 && sum) atomicAdd(sb + ex, (unsigned long long)sum);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += blockDim.x)
    if (sb[t]) atomicAdd(bk + t, sb[t]);
}

// a10: labels of this rank's rows
// One row per lane: a core row's label is comp[v] (the common case); the
// warp's non-core rows (ballot) are then scanned cooperatively, kLabelG lanes
// per row and 4 entries per lane and step, so a scan (at most M-1 entries within
// eps, then the first one beyond) is read as 64-byte coalesced pieces instead of
// a serial per-thread walk.  The first event in column order decides: an entry
// beyond eps ends the scan (noise), a core neighbour within eps gives the label.
constexpr int kLabelG = 4;
template <bool VEC>
__global__ void k_label(const int32_t* __restrict__ nbr, const float* __restrict__ dist, int64_t n_rows,
                        int32_t k, float eps, int64_t row_begin, int64_t N,
                        const uint32_t* __restrict__ bits, const int32_t* __restrict__ comp,
                        int32_t* __restrict__ labels) {
  constexpr int G = kLabelG, RPS = 32 / G;  // rows per cooperative step
  const int lane = threadIdx.x & 31, sub = lane & (G - 1);
  const unsigned gmask = ((1u << G) - 1u) << (lane & ~(G - 1));
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * 32; base < n_rows; base += nwarps * 32) {  // warp-uniform
    const int64_t i = base + lane;
    bool pending = false;
    if (i < n_rows) {
      const int64_t v = row_begin + i;
      if (is_core(bits, v)) labels[i] = comp[v];
      else pending = true;
    }
    unsigned todo = __ballot_sync(0xffffffffu, pending);
    while (todo) {  // RPS non-core rows of this warp at a time, G lanes each
      const int slot = lane / G;
      unsigned t = todo;
      for (int s2 = 0; s2 < slot && t; ++s2) t &= t - 1;  // the slot-th pending row
      const int r = t ? __ffs(t) - 1 : -1;
      for (int s2 = 0; s2 < RPS && todo; ++s2) todo &= todo - 1;
      if (r < 0) continue;  // the whole group idles this step
      const int64_t ii = base + r;
      const int32_t* nr = nbr + ii * k;
      const float* dr = dist + ii * k;
      int32_t lab = -1;
      bool decided = false;
      for (int c0 = 0; c0 < k && !decided; c0 += 4 * G) {
        const int c = c0 + 4 * sub;
        int32_t J[4];
        float w[4];
        if (VEC && c + 4 <= k) {
          const int4 j4 = __ldcs(reinterpret_cast<const int4*>(nr + c));
          const float4 w4 = __ldcs(reinterpret_cast<const float4*>(dr + c));
          J[0] = j4.x; J[1] = j4.y; J[2] = j4.z; J[3] = j4.w;
          w[0] = w4.x; w[1] = w4.y; w[2] = w4.z; w[3] = w4.w;
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const bool in = c + j < k;
            J[j] = in ? __ldcs(nr + c + j) : -1;
            w[j] = in ? __ldcs(dr + c + j) : __int_as_float(0x7f800000);
          }
        }
        int ev = 4;
        bool hit = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (ev < 4) continue;
          if (c + j >= k) { ev = j; break; }  // row end: as beyond eps
          if (!(w[j] <= eps)) { ev = j; continue; }
          const int64_t Jj = J[j];
          if (Jj >= 0 && Jj < N && is_core(bits, Jj)) { ev = j; hit = true; lab = (int32_t)Jj; }
        }
        const unsigned any = __ballot_sync(gmask, ev < 4) & gmask;
        if (any) {
          decided = true;
          if (lane == __ffs(any) - 1) labels[ii] = hit ? comp[lab] : -1;
        }
      }
      if (!decided && sub == 0) labels[ii] = -1;
    }
  }
}

