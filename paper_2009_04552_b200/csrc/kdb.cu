// kdb.cu -- B200-native (sm_100a) kNN-DBSCAN clustering stage behind the C-ABI
// declared in include/kdb.h.
//
// Hot path, one CUDA kernel per step:
//   a1 k_core_mark      core(v) = D[v][M-1] <= eps                 Alg. 1 l.4
//   a2 k_init_*         dense component ids, head pointers L[i]    Alg. 2 l.2-3
//   a3 k_offer_rows     per-vertex first leaving entry -> 64-bit   Alg. 2 l.6-10 + Alg. 3
//                       packed key atomicMin into Kc[comp]          Findmin/pwrite (PAPER.md:562-567,
//                                                                    609-633)
//   a4 k_tie            b tie-break atomicMin into Bc[comp]        reading #6 (paper silent)
//   a5 k_hook           break symmetry + MSF emit                  Alg. 2 l.13-18
//   a6 k_jump/k_relabel pointer jumping, dense renumber, relabel   Alg. 2 l.19-33
//   a7 head pointers    edges that became intra never revive       L[i]
//   a8 termination      no component offers a leaving edge
//   a9 k_canon          label = min core id of the component       north_star
//   a10 k_label         border: first core entry within eps        ClusterBorder
//   a11 k_wbuckets      exact fp64 MSF weight                       north_star
//
// Undirected semantics (reading #4): an entry u->v is an edge of v as well.
//   * KDB_GRAPH_EXACT: an unmirrored in-edge of v weighs >= D[v][k-1] =: kth(v).
//     A component C only hooks when its best row offer is strictly lighter than
//     min_{z in C} kth'(z) (certificate); otherwise it abstains this round (a
//     selected edge is then still the true minimum, so Boruvka stays exact).  If
//     a round would make no progress, a full edge-centric "sweep round" offers
//     every leaving entry to both endpoint components.
//   * otherwise: in-edge lists (transpose of the local candidate entries) are
//     materialised once and scanned alongside the rows every round.
// Multi-GPU (§8(e)): rows are contiguous ranges; per-component arrays are
// replicated; each round all-reduces Kc (u64 MIN) and Bc (u32 MIN) with NCCL,
// then every rank runs hook / jump / relabel identically.
//
// THIS FILE SHARES NO CODE WITH oracle/ (the CPU checker) and never calls it.

#include "kdb.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

// ============================================================================
// error plumbing
// ============================================================================
namespace {

thread_local std::string g_err;
thread_local double g_stats[20];

kdb_status set_err(kdb_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define KDB_CUDA(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return set_err(KDB_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                     __FILE__, __LINE__);                                                \
  } while (0)

#define KDB_TRY(expr)                 \
  do {                                \
    kdb_status s_ = (expr);           \
    if (s_ != KDB_OK) return s_;      \
  } while (0)

constexpr uint64_t kSent = ~0ull;      // sentinel key (reading #11)
constexpr uint32_t kSentB = ~0u;
constexpr uint32_t kInfBits = 0x7f800000u;
constexpr int kThreads = 256;

inline int grid_for(int64_t n, int per_block = kThreads) {
  int64_t g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > (1 << 30)) g = 1 << 30;
  return (int)g;
}

// Grid-stride kernels run exactly one resident wave: min(requested, resident
// CTAs per SM x SMs), from the occupancy calculator (cached per kernel).  A
// second wave would only start after the first finished ALL its strides.
int resident_cap(const void* kern, int block) {
  static std::vector<std::pair<const void*, int>> cache;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  for (auto& e : cache)
    if (e.first == kern) return e.second;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
  const int cap = per_sm * sms;
  cache.emplace_back(kern, cap);
  return cap;
}

// ============================================================================
// launch accounting + optional per-kernel device timing (bench.py's roofline)
// ============================================================================
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
struct Prof {
  bool on = false;
  long long launches = 0;
  std::vector<ProfRec> pending;
  std::vector<cudaEvent_t> pool;
  std::vector<std::string> names;
  std::vector<double> ms;
  std::vector<long long> cnt;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void add(const char* n, double t) {
    for (size_t i = 0; i < names.size(); ++i)
      if (names[i] == n) { ms[i] += t; cnt[i] += 1; return; }
    names.push_back(n);
    ms.push_back(t);
    cnt.push_back(1);
  }
  // resolve recorded pairs (caller synchronised the stream)
  void drain() {
    for (auto& r : pending) {
      float t = 0;
      cudaEventSynchronize(r.b);
      cudaEventElapsedTime(&t, r.a, r.b);
      add(r.name, t);
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    pending.clear();
  }
};
Prof g_prof;
const int g_trace = getenv("KDB_TRACE") ? atoi(getenv("KDB_TRACE")) : 0;  // per-round log to stderr

struct LaunchScope {
  const char* name;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  LaunchScope(const char* n, cudaStream_t s, bool count = true) : name(n), st(s) {
    if (count) ++g_prof.launches;
    if (g_prof.on) {
      a = g_prof.get();
      b = g_prof.get();
      cudaEventRecord(a, st);
    }
  }
  ~LaunchScope() {
    if (g_prof.on) {
      cudaEventRecord(b, st);
      g_prof.pending.push_back({name, a, b});
    }
  }
};
// LAUNCH(kernel, grid, block, stream, args...) -- every kernel of the hot path
#define LAUNCH(kern, grid, block, st, ...)                                          \
  do {                                                                              \
    LaunchScope ls_(#kern, st);                                                     \
    const int g_ = std::min<int>((grid), resident_cap((const void*)(kern), (block))); \
    kern<<<g_, (block), 0, (st)>>>(__VA_ARGS__);                                    \
  } while (0)

// LAUNCH_DYN: the same with dynamic shared memory (opt-in above 48 KB)
int resident_cap_smem(const void* kern, int block, size_t smem) {
  static std::vector<std::pair<const void*, int>> cache;
  for (auto& e : cache)
    if (e.first == kern) return e.second;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms = 148, dev = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  cache.emplace_back(kern, per_sm * sms);
  return per_sm * sms;
}
#define LAUNCH_DYN(kern, grid, block, smem, st, ...)                                           \
  do {                                                                                         \
    LaunchScope ls_(#kern, st);                                                                \
    const int g_ = std::min<int>((grid), resident_cap_smem((const void*)(kern), (block), (smem))); \
    kern<<<g_, (block), (smem), (st)>>>(__VA_ARGS__);                                          \
  } while (0)

// ============================================================================
// NCCL (dlopen, so libkdb.so loads without NCCL on the path)
// ============================================================================
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

kdb_status nccl_load() {
  if (g_nccl.h) return KDB_OK;
  const char* path = getenv("KDB_NCCL_LIBRARY");
  void* h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) return set_err(KDB_ENCCL, "cannot dlopen NCCL (%s): %s", path ? path : "libnccl.so.2", dlerror());
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.AllReduce || !g_nccl.CommDestroy)
    return set_err(KDB_ENCCL, "NCCL library lacks required symbols");
  g_nccl.h = h;
  return KDB_OK;
}

}  // namespace

struct kdb_comm {
  int kind = 0;  // 1 = nccl, 2 = sim
  int rank = 0, nranks = 1;
  ncclComm_t nccl = nullptr;
};

namespace {

kdb_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return KDB_OK;
  return set_err(KDB_ENCCL, "%s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
}

// ============================================================================
// device helpers
// ============================================================================
__device__ __forceinline__ uint32_t mono_bits(float w) {
  uint32_t u = __float_as_uint(w);
  return u == 0x80000000u ? 0u : u;  // -0 -> +0 (reading #6)
}

__device__ __forceinline__ bool is_core(const uint32_t* __restrict__ bits, int64_t v) {
  return (__ldcg(bits + (v >> 5)) >> (v & 31)) & 1u;
}

// Random 4/8-byte gathers go through ld.global.cg (L2 only, 32-B sector
// requests).  The read-only .nc path (LDG.CONSTANT) promoted each miss to a
// whole 128-B line: 4x the L2/DRAM traffic for a 4-B gather.
template <typename T>
__device__ __forceinline__ T gat(const T* p) { return __ldcg(p); }

// atomicMin preceded by a plain read: an offer that cannot lower the current
// key issues no atomic (same-address atomics serialise at the L2 slice when
// many rows offer to one component).  A stale read only lets an atomic through.
__device__ __forceinline__ void min_offer(unsigned long long* p, unsigned long long x) {
  if (x < __ldcg(p)) atomicMin(p, x);
}

__device__ __forceinline__ uint64_t pack_key(uint32_t wbits, uint32_t a) {
  return ((uint64_t)wbits << 32) | a;
}

struct RoundCounters {
  uint32_t msf_count;            // edges emitted so far (all rounds)
  uint32_t pad0;
  uint32_t hooks;                // this round
  uint32_t offered;              // components with a finite key
  uint32_t uncertified;          // offered but abstaining (exact-mode certificate)
  uint32_t n_roots;              // components after contraction
  uint32_t n_act[2];             // per-rank scratch (row / in active counts), see host
  uint32_t n_off;
  uint32_t violation;            // a hook target's key exceeds the hooker's: the
                                 // KDB_GRAPH_EXACT promise was false (or a bug)
  uint32_t n_cont;               // rows continuing in the warp-per-row scan
  uint32_t pad1;
  uint32_t grab;                 // chunk cursor of the ordered row kernels (per rank)
  uint32_t n_off2;
  uint32_t na[2];                // per rank: row-list sizes, ping-pong (input na[cur], output na[cur^1])
  uint32_t ni[2];                // per rank: in-list sizes, ping-pong
  long long Cs[2];               // global: component count, ping-pong (current Cs[par], next Cs[par^1])
  unsigned long long entries;    // graph entries (id + weight) read by offer kernels
};

// block-aggregated slot reservation: ONE global atomic per block and call.
// Must be reached by every thread of the block (block-uniform control flow).
__device__ __forceinline__ uint32_t block_reserve(uint32_t* counter, bool want) {
  __shared__ uint32_t s_cnt[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (lane == 0) s_cnt[warp] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int w = 0; w < nw; ++w) { const uint32_t c = s_cnt[w]; s_cnt[w] = tot; tot += c; }
    s_cnt[32] = tot ? atomicAdd(counter, tot) : 0u;
  }
  __syncthreads();
  const uint32_t slot = s_cnt[32] + s_cnt[warp] + __popc(m & ((1u << lane) - 1u));
  __syncthreads();
  return slot;
}

// block-aggregated counter increment (block-uniform call)
__device__ __forceinline__ void block_count(uint32_t* counter, bool pred) {
  __shared__ uint32_t s_c;
  if (threadIdx.x == 0) s_c = 0;
  __syncthreads();
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(&s_c, (uint32_t)__popc(m));
  __syncthreads();
  if (threadIdx.x == 0 && s_c) atomicAdd(counter, s_c);
  __syncthreads();
}

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
                                   uint32_t* __restrict__ kmin, const int64_t* __restrict__ Cp = nullptr) {
  if (Cp) C = *Cp;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
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

struct RowScan {
  bool found;
  int h;          // new head: the first leaving entry, or k when exhausted
  uint64_t best;  // minimum key of the group
  uint32_t bestb;
  int32_t bestc;  // component of the best entry's far endpoint
};

// Scan row (nr, dr) of vertex v (component cv) from head h.  direct: singleton
// components (round 1, exact mode) -- every candidate leaves; with all_core the
// dense component id of a vertex is the vertex itself (no gathers at all).
template <bool VEC, bool DIRECT>
__device__ __forceinline__ RowScan scan_row(const int32_t* __restrict__ nr, const float* __restrict__ dr, int k,
                                            float eps, int32_t v, int32_t cv, int h, int64_t N,
                                            const int32_t* __restrict__ comp, int all_core,
                                            unsigned long long& reads) {
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
      cj[j] = cand ? ((DIRECT && all_core) ? J[j] : gat(comp + J[j])) : -1;
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
                                                   int4* __restrict__ rec1) {
  __shared__ __align__(16) Rec s_rec[kChunk];
  __shared__ uint32_t s_n, s_chunk, s_base;
  for (;;) {
    if (threadIdx.x == 0) { s_chunk = atomicAdd(grab, 1u); s_n = 0; }
    __syncthreads();
    const int64_t base = (int64_t)s_chunk * kChunk;
    if (base >= n_rows) break;
    for (int t = 0; t < kChunk; t += 256) {
      const int64_t i = base + t + threadIdx.x;
      if (i >= n_rows) continue;
      const int64_t v = row_begin + i;
      const int32_t cv = comp[v];
      if (cv < 0) continue;
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
        kmin[cv] = kb;
      }
      int4* o = LE + i * (kW / 2);
#pragma unroll
      for (int q = 0; q < kW / 2; ++q)
        __stcs(o + q, make_int4(J[2 * q], __float_as_int(w[2 * q]), J[2 * q + 1], __float_as_int(w[2 * q + 1])));
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
#pragma unroll
      for (int c = 0; c < kW; ++c) {
        if (done || c >= k) continue;
        const int32_t Jc = J[c];
        if (!r.found) {
          if (!(w[c] <= eps)) { done = true; continue; }  // sorted: no candidate at all
          if (Jc < 0 || Jc >= N || Jc == v) continue;
          const int32_t cc = all_core ? Jc : gat(comp + Jc);
          if (cc < 0) continue;
          r.found = true;
          r.h = c;
          wstar = w[c];
          r.best = pack_key(mono_bits(w[c]), (uint32_t)min(v, (int64_t)Jc));
          r.bestb = (uint32_t)max(v, (int64_t)Jc);
          r.bestc = cc;
        } else {
          if (w[c] != wstar) { done = true; continue; }
          if (Jc < 0 || Jc >= N || Jc == v) continue;
          const int32_t cc = all_core ? Jc : gat(comp + Jc);
          if (cc < 0) continue;
          const uint64_t kk = pack_key(mono_bits(w[c]), (uint32_t)min(v, (int64_t)Jc));
          const uint32_t bb = (uint32_t)max(v, (int64_t)Jc);
          if (kk < r.best || (kk == r.best && bb < r.bestb)) { r.best = kk; r.bestb = bb; r.bestc = cc; }
        }
      }
      if (!done && k > kW) {  // the search or the tie group runs past the ELL: scan the row in place
        unsigned long long rd = 0;
        r = scan_row<false, true>(nr, dr, k, eps, (int32_t)v, -1, 0, N, comp, all_core, rd);
      }
      if (rec1) {  // single rank: one packed record per component for k_hook<true>
        __stcg(rec1 + cv, make_int4((int)(uint32_t)r.best, (int)(uint32_t)(r.best >> 32), (int)r.bestb, (int)kb));
        if (r.found) tgt[cv] = r.bestc;
      } else if (r.found) {
        Kc[cv] = r.best;
        Bc[cv] = r.bestb;
        tgt[cv] = r.bestc;
      }
      if (r.found) s_rec[atomicAdd(&s_n, 1u)] = Rec{(int32_t)v, r.h};
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_n ? atomicAdd(n_act, s_n) : 0u;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < s_n; j += blockDim.x) act[s_base + j] = s_rec[j];
    __syncthreads();
  }
}



// Scan row v (component cv) from head h: columns < kW from the ELL row, the
// rest (rare: a candidate prefix longer than kW) from the graph row.  DIRECT:
// singleton components (round 1, exact mode), every candidate leaves; with
// all_core a vertex's dense component id is the vertex itself (no gathers).
// GW: component gathers are issued GW entries at a time; once the minimum is
// found only entries of its weight (decided from the loaded w) are gathered,
// so a smaller GW trades memory-level parallelism for L2 sector traffic.
template <bool DIRECT, int GW = 4>
__device__ __forceinline__ RowScan scan_ell(const int4* __restrict__ le, const int32_t* __restrict__ nr,
                                            const float* __restrict__ dr, int k, float eps, int32_t v, int32_t cv,
                                            int h, int64_t N, const int32_t* __restrict__ comp, int all_core,
                                            unsigned long long& reads) {
  RowScan r{false, k, kSent, kSentB, -1};
  uint32_t wstar = 0;
  const int kend = min(k, kW);
  int c0 = h & ~3;
  bool done = false;
  while (!done && c0 < kend) {
    int4 p0, p1;
    ld256cs(le + (c0 >> 1), p0, p1);
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
      bool cand = idx >= h && idx < kend && w[j] <= eps && J[j] >= 0 && J[j] < N && J[j] != v;
      if (GW < 4 && r.found && mono_bits(w[j]) != wstar) cand = false;  // past the tie group: no gather
      cj[j] = cand ? ((DIRECT && all_core) ? J[j] : gat(comp + J[j])) : -1;
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
      } else {
        if (wb != wstar) { done = true; continue; }
        if (!leaving) continue;
        const uint64_t kk = pack_key(wb, (uint32_t)min(v, J[j]));
        const uint32_t bb = (uint32_t)max(v, J[j]);
        if (kk < r.best || (kk == r.best && bb < r.bestb)) { r.best = kk; r.bestb = bb; r.bestc = cj[j]; }
      }
    }
    }
    c0 += 4;
  }
  if (!done && k > kW) {
    // the candidate prefix (or the minimum's tie group) runs past the ELL
    if (!r.found) {
      RowScan t = scan_row<false, DIRECT>(nr, dr, k, eps, v, cv, max(h, kW), N, comp, all_core, reads);
      return t;
    }
    // continue the tie group of weight wstar in the graph row
    for (int c = kW; c < k; ++c) {
      const float wc = __ldcg(dr + c);
      if (mono_bits(wc) != wstar || !(wc <= eps)) break;
      const int32_t Jc = __ldcg(nr + c);
      ++reads;
      if (Jc < 0 || Jc >= N || Jc == v) continue;
      const int32_t cc = (DIRECT && all_core) ? Jc : gat(comp + Jc);
      if (cc < 0 || (!DIRECT && cc == cv)) continue;
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
__global__ void __launch_bounds__(256) k_light_first(const int4* __restrict__ LE, const int32_t* __restrict__ nbr,
                                                     const float* __restrict__ dist, int32_t ld, int32_t k, float eps,
                                                     int64_t row_begin, int64_t N, const int32_t* __restrict__ comp,
                                                     int all_core, const Rec* __restrict__ act, uint32_t n_in,
                                                     Rec* __restrict__ act_out, uint32_t* __restrict__ n_out,
                                                     uint32_t* __restrict__ grab,
                                                     uint64_t* __restrict__ Kc, uint32_t* __restrict__ Bc,
                                                     int32_t* __restrict__ tgt, unsigned long long* __restrict__ n_entries, const uint32_t* __restrict__ n_in_p = nullptr) {
  if (n_in_p) n_in = *n_in_p;
  __shared__ __align__(16) Rec s_rec[kChunk];
  __shared__ uint32_t s_n, s_chunk, s_base;
  unsigned long long reads = 0;
  for (;;) {
    if (threadIdx.x == 0) { s_chunk = atomicAdd(grab, 1u); s_n = 0; }
    __syncthreads();
    const uint64_t base = (uint64_t)s_chunk * kChunk;
    if (base >= n_in) break;
    for (int t = 0; t < kChunk; t += 256) {
      const uint64_t s = base + t + threadIdx.x;
      if (s >= n_in) continue;
      const int2 a = __ldcs(reinterpret_cast<const int2*>(act + s));
      const int32_t v = a.x;
      const int64_t i = (int64_t)v - row_begin;
      const RowScan r = scan_ell<true>(LE + i * (kW / 2), nbr + i * ld, dist + i * ld, k, eps, v, -1, a.y, N, comp,
                                       all_core, reads);
      if (r.found) {
        const int32_t cv = all_core ? v : gat(comp + v);
        Kc[cv] = r.best;
        Bc[cv] = r.bestb;
        tgt[cv] = r.bestc;
        s_rec[atomicAdd(&s_n, 1u)] = Rec{v, r.h};
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

// later rounds over the ELL; see k_offer_round
template <int GW>
__global__ void __launch_bounds__(256) k_light_round(const int4* __restrict__ LE, const int32_t* __restrict__ nbr,
                                                     const float* __restrict__ dist, int32_t ld, int32_t k, float eps,
                                                     int64_t row_begin, int64_t N, const int32_t* __restrict__ comp,
                                                     const Rec* __restrict__ act, uint32_t n_in,
                                                     Rec* __restrict__ act_out, uint32_t* __restrict__ n_out,
                                                     uint32_t* __restrict__ grab, Offer* __restrict__ offers,
                                                     unsigned long long* __restrict__ Kc,
                                                     unsigned long long* __restrict__ n_entries, const uint32_t* __restrict__ n_in_p = nullptr,
                                                     int precheck = 0) {
  if (n_in_p) n_in = *n_in_p;
  __shared__ __align__(16) Rec s_rec[kChunk];
  __shared__ __align__(16) Offer s_off[kChunk];
  __shared__ uint32_t s_n, s_chunk, s_base;
  unsigned long long reads = 0;
  for (;;) {
    if (threadIdx.x == 0) { s_chunk = atomicAdd(grab, 1u); s_n = 0; }
    __syncthreads();
    const uint64_t base = (uint64_t)s_chunk * kChunk;
    if (base >= n_in) break;
    for (int t = 0; t < kChunk; t += 256) {
      const uint64_t s = base + t + threadIdx.x;
      if (s >= n_in) continue;
      const int2 a = __ldcs(reinterpret_cast<const int2*>(act + s));
      const int32_t v = a.x;
      const int32_t cv = gat(comp + v);
      const int64_t i = (int64_t)v - row_begin;
      const RowScan r = scan_ell<false, GW>(LE + i * (kW / 2), nbr + i * ld, dist + i * ld, k, eps, v, cv, a.y, N,
                                            comp, 0, reads);
      if (r.found) {
        if (precheck) min_offer(Kc + cv, (unsigned long long)r.best);
        else atomicMin(Kc + cv, (unsigned long long)r.best);
        const uint32_t j = atomicAdd(&s_n, 1u);
        s_rec[j] = Rec{v, r.h};
        s_off[j] = Offer{cv, r.bestb, r.best};
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_n ? atomicAdd(n_out, s_n) : 0u;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < s_n; j += blockDim.x) {
      __stcs(reinterpret_cast<int2*>(act_out + s_base + j), *reinterpret_cast<const int2*>(s_rec + j));
      __stcs(reinterpret_cast<int4*>(offers + s_base + j), *reinterpret_cast<const int4*>(s_off + j));
    }
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
                       const int4* __restrict__ rec1) {
  if (Cp) C = *Cp;
  __shared__ uint64_t s_key[kHookChunk];
  __shared__ uint32_t s_w[kHookChunk];
  __shared__ uint32_t s_n, s_base;
  uint32_t n_off = 0, n_unc = 0, n_hook = 0;
  for (int64_t chunk = blockIdx.x; chunk * kHookChunk < C; chunk += gridDim.x) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int t = 0; t < kHookChunk; t += blockDim.x) {
      const int64_t c = chunk * kHookChunk + t + threadIdx.x;
      if (c >= C) continue;
      uint64_t K;
      uint32_t Bown = 0, kbown = kInfBits;
      if (PACKED) {  // round 1, single rank: (K, B, kmin) of a component in one 16-B record
        const int4 q = __ldcs(rec1 + c);
        K = (uint64_t)(uint32_t)q.x | ((uint64_t)(uint32_t)q.y << 32);
        Bown = (uint32_t)q.z;
        kbown = (uint32_t)q.w;
      } else {
        K = Kc[c];
      }
      int32_t p = (int32_t)c;
      if (K != kSent) {
        ++n_off;
        if (PACKED ? !((uint32_t)(K >> 32) < kbown) : !certified(K, kmin, c)) {
          ++n_unc;
        } else {
          const uint32_t a = (uint32_t)K;
          const uint32_t b = PACKED ? Bown : Bc[c];
          int32_t t2;
          if (tgt) {
            t2 = tgt[c];
          } else {
            const int32_t x = (gat(comp + a) == (int32_t)c) ? (int32_t)b : (int32_t)a;
            t2 = gat(comp + x);
          }
          bool mutual, cert_t = true;
          if (PACKED) {  // one random 16-B read of the target's record
            const int4 q = __ldcg(rec1 + t2);
            const uint64_t Kt = (uint64_t)(uint32_t)q.x | ((uint64_t)(uint32_t)q.y << 32);
            const uint32_t Bt = (uint32_t)q.z;
            cert_t = Kt != kSent && (uint32_t)(Kt >> 32) < (uint32_t)q.w;
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
                       const int64_t* __restrict__ Cp = nullptr) {
  if (Cp) C = *Cp;
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
    rootof[c] = x;
  }
}

__global__ void k_root_flags(int64_t C, const int32_t* __restrict__ rootof, int32_t* __restrict__ flag,
                             const int64_t* __restrict__ Cp = nullptr) {
  // C is the (host) upper bound the scan runs over; with Cp the true count is
  // on the device and the flags beyond it are 0
  const int64_t Ct = Cp ? *Cp : C;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x)
    flag[c] = c < Ct && rootof[c] == (int32_t)c;
}

// number of roots = new component count, from the exclusive scan
__global__ void k_count_roots(const int64_t* __restrict__ Cp, const int32_t* __restrict__ newid,
                              const int32_t* __restrict__ flag, int64_t* __restrict__ Cn) {
  const int64_t C = *Cp;
  *Cn = C > 0 ? (int64_t)newid[C - 1] + flag[C - 1] : 0;
}

// new per-component arrays: cmin/kmin are minima over the merged tree
__global__ void k_merge(int64_t C, const int32_t* __restrict__ rootof, const int32_t* __restrict__ newid,
                        const int32_t* __restrict__ cmin, const uint32_t* __restrict__ kmin,
                        int32_t* __restrict__ cmin2, uint32_t* __restrict__ kmin2, int32_t* __restrict__ map, const int64_t* __restrict__ Cp = nullptr) {
  if (Cp) C = *Cp;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = newid ? gat(newid + rootof[c]) : rootof[c];  // sparse ids: the root itself
    map[c] = r;
    atomicMin(cmin2 + r, cmin[c]);
    if (kmin) {
      const uint32_t km = kmin[c];
      if (km != kInfBits) atomicMin(kmin2 + r, km);  // kmin2 starts at +inf
    }
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
__global__ void k_msf_unpack(int64_t m, const uint32_t* __restrict__ ka, const unsigned long long* __restrict__ vb,
                             uint32_t* __restrict__ b, float* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t ai = ka[i];
    if (i > 0 && ka[i - 1] == ai) continue;  // not the start of a run
    int64_t j = i + 1;
    while (j < m && ka[j] == ai) ++j;
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
constexpr int kFilterThreads = KDB_FILTER_THREADS;  // rows per tile = threads per block
constexpr int kFilterUnroll = KDB_FILTER_UNROLL;    // 16-B id chunks in flight per thread
constexpr size_t kFilterSmem = kBloomBits / 8;

// Blocked Bloom filter: key x selects ONE 32-bit word (top 15 bits of x*C1)
// and sets 3 bits in it (three 5-bit fields of x*C2): a single shared-memory
// probe per test, false-positive rate ~1e-4 at ~2e4 keys.
// One multiplicative hash h = x * phi serves both: the word from its top 15
// bits, the three bit positions from bits [0,5), [5,10), [10,15) (the low bits
// of h are a bijection of the low bits of x, independent of the word choice).
// 1 << (s & 31) is one funnel shift (SHF.L.W wraps the amount).
__device__ __forceinline__ uint32_t bloom_hash(uint32_t x) { return x * 0x9E3779B1u; }
__device__ __forceinline__ uint32_t bloom_word_h(uint32_t h) { return h >> 17; }
__device__ __forceinline__ uint32_t bloom_mask_h(uint32_t h) {
  return __funnelshift_l(0u, 1u, h) | __funnelshift_l(0u, 1u, h >> 5) | __funnelshift_l(0u, 1u, h >> 10);
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

// The filter: every rank streams its rows once, in tiles of kFilterThreads
// rows.  Per tile, thread i stages row i's data in shared memory (comp[v] and
// the id range of comp[v]); then the tile's R*k ids are swept in flat order,
// VEC per thread and step.  Fast path: J inside the id range of comp[v] and
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
template <int VEC, bool FAST, bool COLS>
__global__ void __launch_bounds__(kFilterThreads) k_filter(
    const int32_t* __restrict__ nbr, const float* __restrict__ dist, int64_t n_rows, int32_t ld, int32_t k, float tau, float eps,
    int64_t row_begin, int64_t N, const int32_t* __restrict__ comp, const int2* __restrict__ rng, const uint32_t* __restrict__ bloom, FastDiv fd,
    HEdge* __restrict__ out, uint32_t cap, uint32_t* __restrict__ n_out, unsigned long long* __restrict__ n_slow) {
  extern __shared__ uint32_t s_bloom[];
  __shared__ FRow s_row[kFilterThreads];
  constexpr int R = kFilterThreads;
  const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(s_bloom);
  if (FAST) {
    for (int t = threadIdx.x; t < kBloomBits / 32; t += blockDim.x) s_bloom[t] = bloom[t];
  }
  const uint32_t Nu = (uint32_t)N;
  const int64_t n_tiles = (n_rows + R - 1) / R;
  uint32_t slow = 0;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t r0 = tile * R;
    const int nr = (int)((n_rows - r0) < R ? (n_rows - r0) : R);
    __syncthreads();  // previous tile's readers are done with s_row (and the Bloom copy is complete)
    if ((int)threadIdx.x < nr) {
      const int64_t i = r0 + threadIdx.x;
      FRow fr;
      fr.cr = __ldg(comp + row_begin + i);
      fr.lo = 0;
      fr.span = 0;
      if (FAST && fr.cr >= 0) {
        const int2 rg = __ldg(rng + fr.cr);
        if (rg.y > rg.x) { fr.lo = (uint32_t)rg.x; fr.span = (uint32_t)(rg.y - rg.x); }
      }
      s_row[threadIdx.x] = fr;
    }
    __syncthreads();
    const int32_t* __restrict__ nt = nbr + r0 * ld;  // this tile's ids (contiguous)
    const float* __restrict__ dt = dist + r0 * ld;
    const uint32_t cpr = (uint32_t)((k + VEC - 1) / VEC);  // COLS: chunks per row
    const uint32_t n_chunks = COLS ? (uint32_t)nr * cpr : (uint32_t)(((int64_t)nr * ld) / VEC);
    // kFilterUnroll chunks per thread and step: their id loads are issued
    // together (the sweep is bound by load latency x loads in flight)
    for (uint32_t base = 0; base < n_chunks; base += blockDim.x * kFilterUnroll) {
      int32_t J[kFilterUnroll][VEC];
#pragma unroll
      for (int t = 0; t < kFilterUnroll; ++t) {
        const uint32_t u = base + t * blockDim.x + threadIdx.x;
        uint32_t off = u;  // chunk offset from the tile start
        if (COLS && u < n_chunks) {
          const uint32_t lr = fd.small ? __umulhi(u, fd.m32) : (uint32_t)fdiv(u, fd);
          off = lr * (uint32_t)(ld / VEC) + (u - lr * cpr);
        }
        if (VEC == 4) {
          const int4 j4 = u < n_chunks ? __ldcs(reinterpret_cast<const int4*>(nt) + off) : make_int4(-1, -1, -1, -1);
          J[t][0] = j4.x; J[t][1] = j4.y; J[t][2] = j4.z; J[t][3] = j4.w;
        } else {
          J[t][0] = u < n_chunks ? __ldcs(nt + off) : -1;
        }
      }
#pragma unroll
      for (int t = 0; t < kFilterUnroll; ++t) {
        const uint32_t u = base + t * blockDim.x + threadIdx.x;
        uint32_t survm = 0, lr = 0, col = 0, off = u;
        int32_t cj[VEC], cr = -1;
        float w[VEC];
        if (u < n_chunks) {
          if (COLS) {
            lr = fd.small ? __umulhi(u, fd.m32) : (uint32_t)fdiv(u, fd);  // row within the tile
            col = (u - lr * cpr) * VEC;
            off = lr * (uint32_t)(ld / VEC) + (u - lr * cpr);
          } else {
            const uint32_t n = u * VEC;
            lr = fd.small ? __umulhi(n, fd.m32) : (uint32_t)fdiv(n, fd);  // row within the tile
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
          const int lane = threadIdx.x & 31;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int x = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += x;
          }
          const int tot = __shfl_sync(0xffffffffu, incl, 31);
          uint32_t base_slot = 0;
          if (lane == 31) base_slot = atomicAdd(n_out, (uint32_t)tot);
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

// ============================================================================
// host side
// ============================================================================
// exact value of sum_e bk[e] * 2^(max(e,1) - 150), rounded once to double
double exact_bucket_sum(const unsigned long long* bk) {
  uint64_t L[7] = {0, 0, 0, 0, 0, 0, 0};  // little-endian limbs, value * 2^149
  for (int e = 0; e < 256; ++e) {
    if (!bk[e]) continue;
    const int sh = (e ? e : 1) - 1;  // 2^(max(e,1)-150) = 2^(sh) * 2^-149
    const int q = sh / 64, r = sh % 64;
    unsigned __int128 add0 = (unsigned __int128)bk[e] << r;  // up to 128 bits
    uint64_t parts[3] = {(uint64_t)add0, (uint64_t)(add0 >> 64), 0};
    unsigned __int128 carry = 0;
    for (int j = q; j < 7; ++j) {
      unsigned __int128 s = (unsigned __int128)L[j] + carry + (j - q < 3 ? parts[j - q] : 0);
      L[j] = (uint64_t)s;
      carry = s >> 64;
    }
  }
  int top = -1;
  for (int j = 6; j >= 0; --j)
    if (L[j]) { top = j * 64 + 63 - __builtin_clzll(L[j]); break; }
  if (top < 0) return 0.0;
  auto bit = [&](int p) -> int { return p < 0 ? 0 : (int)((L[p / 64] >> (p % 64)) & 1u); };
  // 53-bit mantissa [top-52, top], round bit top-53, sticky below
  uint64_t man = 0;
  for (int p = top; p > top - 53; --p) man = (man << 1) | (uint64_t)bit(p);
  const int rb = bit(top - 53);
  bool sticky = false;
  for (int p = top - 54; p >= 0 && !sticky; --p) sticky = bit(p);
  if (rb && (sticky || (man & 1u))) ++man;  // round to nearest even
  return ldexp((double)man, top - 52 - 149);
}

// heavy-phase survivor capacity per rank (edges); beyond it kdb_mst falls back
// to plain rows-Boruvka over the whole candidate graph (still exact)
constexpr int kTauSamples = 8192;
inline int64_t survivor_cap(int64_t n_rows, int64_t k) {
  return std::max<int64_t>(n_rows / 4, std::min<int64_t>(n_rows * k / 4, (int64_t)1 << 24)) + 65536;
}

struct Carver {
  char* base;
  size_t off = 0, cap;
  bool dry;
  template <typename T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = dry ? nullptr : reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    return p;
  }
};

struct RankState {
  int64_t row_begin = 0, n_rows = 0;
  const int32_t* nbr = nullptr;
  const float* dist = nullptr;
  Rec* act[2] = {nullptr, nullptr};  // active rows (v, head), ping-pong
  uint32_t n_act = 0;                 // live rows in act[cur]
  bool compact = false;               // rows phase reads the light ELL (else the graph rows)
  int4* LE = nullptr;                 // light ELL [n_rows][kW] (J, w bits) pairs
  // offers: [0, n_rows) from rows (same slot as the row's next record),
  // [n_rows, n_rows + N) from in-lists (general mode)
  Offer* offers = nullptr;
  int64_t off_cap_rows = 0;
  // per-rank partial Kc/Bc (sim ranks > 0) -- else alias the shared ones
  uint64_t* Kc = nullptr;
  uint32_t* Bc = nullptr;
  int32_t* tgt = nullptr;
  // in-edge lists (general mode)
  unsigned long long* in_off = nullptr;
  int32_t* in_len = nullptr;
  int32_t* in_src = nullptr;
  float* in_w = nullptr;
  int32_t* in_act[2] = {nullptr, nullptr};
  uint32_t n_in_act = 0;
  RoundCounters* ctr = nullptr;  // per-rank counters (act/off)
  // heavy phase: survivors (ping-pong) and their keep flags
  HEdge* hs[2] = {nullptr, nullptr};
  uint8_t* hkeep = nullptr;
  uint32_t hs_cap = 0, n_hs = 0;
  uint32_t* n_hs_dev = nullptr;  // [2]: filter count, compaction count
};

struct Layout {
  // shared
  uint32_t* woff;
  int32_t *cmin, *cmin2, *parent, *rootof, *newid, *flag;
  uint32_t *kmin, *kmin2;
  uint64_t* Kc;
  uint32_t* Bc;
  int32_t* tgt;
  int all_core = 0;
  uint64_t* e_key;
  float* e_w;
  unsigned long long* buckets;
  int4* rec1;       // round 1, single rank, exact mode: packed (K, B, kmin) per component
  int32_t* hcomp;   // heavy phase: light component -> heavy component
  int32_t* dom;     // filter fast path: dominant component per id block
  uint32_t* bloom;  // filter fast path: Bloom filter of the exceptions
  unsigned long long* fcount;  // [0] exceptions, [1] slow-path entries
  float* tau_sample;
  RoundCounters* ctr;
  void* cub_tmp;
  size_t cub_bytes;
  std::vector<RankState> ranks;
};

size_t cub_tmp_bytes(int64_t N, int64_t cap_edges) {
  size_t a = 0, b = 0, c = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (const int32_t*)nullptr, (int32_t*)nullptr, (int)std::max<int64_t>(N + 1, 1));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const unsigned long long*)nullptr,
                                (unsigned long long*)nullptr, (int)std::max<int64_t>(N + 1, 1));
  cub::DeviceRadixSort::SortPairs(nullptr, c, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (int)std::max<int64_t>(cap_edges, 1));
  size_t f = 0;
  size_t h3 = 0;
  cub::DeviceSelect::Flagged(nullptr, h3, (const HEdge*)nullptr, (const uint8_t*)nullptr, (HEdge*)nullptr,
                             (uint32_t*)nullptr, (int)std::min<int64_t>(survivor_cap(N, 65535) + 1, INT32_MAX));
  f = std::max(f, h3);
  return std::max(std::max(a, f), std::max(b, c)) + 256;
}

// carve the workspace; returns bytes needed
size_t carve(Layout& L, char* base, bool dry, int64_t N, int nr, const int64_t* rb, const int64_t* rn,
             bool general, int32_t k, int64_t hs_cap_override = -1) {
  Carver cv{base, 0, 0, dry};
  const int64_t nwords = (N + 31) / 32;
  L.woff = cv.take<uint32_t>(nwords + 1);
  L.cmin = cv.take<int32_t>(N + 1);
  L.cmin2 = cv.take<int32_t>(N + 1);
  L.parent = cv.take<int32_t>(N + 1);
  L.rootof = cv.take<int32_t>(N + 1);
  L.newid = cv.take<int32_t>(N + 1);
  L.flag = cv.take<int32_t>(N + 1);
  L.kmin = cv.take<uint32_t>(N + 1);
  L.kmin2 = cv.take<uint32_t>(N + 1);
  L.Kc = cv.take<uint64_t>(N + 1);
  L.Bc = cv.take<uint32_t>(N + 1);
  L.tgt = cv.take<int32_t>(N + 1);
  L.e_key = cv.take<uint64_t>(N + 1);
  L.e_w = cv.take<float>(N + 1);
  L.buckets = cv.take<unsigned long long>(256);
  L.rec1 = general ? nullptr : cv.take<int4>(N + 1);
  L.hcomp = cv.take<int32_t>(N + 1);
  L.dom = cv.take<int32_t>(kDomMax);
  L.bloom = cv.take<uint32_t>(kBloomBits / 32);
  L.fcount = cv.take<unsigned long long>(2);
  L.tau_sample = cv.take<float>(kTauSamples);
  L.ctr = cv.take<RoundCounters>(1);
  L.cub_bytes = cub_tmp_bytes(N, N + 1);
  L.cub_tmp = cv.take<char>(L.cub_bytes);
  L.ranks.assign(nr, RankState());
  for (int r = 0; r < nr; ++r) {
    RankState& R = L.ranks[r];
    R.row_begin = rb[r];
    R.n_rows = rn[r];
    const int64_t n = std::max<int64_t>(rn[r], 1);
    R.act[0] = cv.take<Rec>(n);
    R.act[1] = cv.take<Rec>(n);
    R.LE = cv.take<int4>(n * (kW / 2));
    R.off_cap_rows = n;
    R.offers = cv.take<Offer>(general ? n + N : n);
    R.ctr = cv.take<RoundCounters>(1);
    if (r > 0) {
      R.Kc = cv.take<uint64_t>(N + 1);
      R.Bc = cv.take<uint32_t>(N + 1);
      R.tgt = cv.take<int32_t>(N + 1);
    } else {
      R.Kc = L.Kc;
      R.Bc = L.Bc;
      R.tgt = L.tgt;
    }
    R.hs_cap = (uint32_t)std::min<int64_t>(hs_cap_override >= 0 ? std::max<int64_t>(hs_cap_override, 1)
                                                                   : survivor_cap(n, k),
                                           (int64_t)UINT32_MAX - 1);
    R.hs[0] = cv.take<HEdge>(R.hs_cap);
    R.hs[1] = cv.take<HEdge>(R.hs_cap);
    R.hkeep = cv.take<uint8_t>(R.hs_cap);
    R.n_hs_dev = cv.take<uint32_t>(2);
    if (general) {
      R.in_off = cv.take<unsigned long long>(N + 1);
      R.in_len = cv.take<int32_t>(N);
      R.in_src = cv.take<int32_t>(n * (int64_t)k);
      R.in_w = cv.take<float>(n * (int64_t)k);
      R.in_act[0] = cv.take<int32_t>(N);
      R.in_act[1] = cv.take<int32_t>(N);
    }
  }
  return cv.off + 256;
}

kdb_status validate_graph(const kdb_graph* g) {
  if (!g) return set_err(KDB_EINVAL, "graph is NULL");
  if (g->n_total < 0 || g->n_total >= (int64_t)INT32_MAX)
    return set_err(KDB_EINVAL, "n_total out of range [0, 2^31-1)");
  if (g->k_max < 1 || g->k_max > 65535) return set_err(KDB_EINVAL, "k_max must be in [1, 65535]");
  if (g->n_rows < 0 || g->row_begin < 0 || g->row_begin + g->n_rows > g->n_total)
    return set_err(KDB_EINVAL, "rank row range outside [0, n_total)");
  if (g->n_rows > 0 && (!g->nbr || !g->dist)) return set_err(KDB_EINVAL, "nbr/dist is NULL");
  if (((uintptr_t)g->nbr & 15u) || ((uintptr_t)g->dist & 15u))
    return set_err(KDB_EINVAL, "nbr/dist must be 16-byte aligned");
  if (g->flags & ~KDB_GRAPH_EXACT) return set_err(KDB_EINVAL, "unknown graph flags");
  if (g->edge_cols < 0 || g->edge_cols > g->k_max) return set_err(KDB_EINVAL, "edge_cols must be in [0, k_max]");
  return KDB_OK;
}

kdb_status validate_eps(float eps) {
  if (!(eps > 0.0f) || !(eps < __builtin_inff())) return set_err(KDB_EINVAL, "eps must be in (0, +inf)");
  return KDB_OK;
}

// rank ranges of the computation this process performs
void rank_ranges(const kdb_graph* g, kdb_comm* comm, std::vector<int64_t>& rb, std::vector<int64_t>& rn) {
  rb.clear();
  rn.clear();
  if (comm && comm->kind == 2) {
    const int P = comm->nranks;
    for (int r = 0; r < P; ++r) {
      const int64_t b = g->n_rows * r / P, e = g->n_rows * (r + 1) / P;
      rb.push_back(g->row_begin + b);
      rn.push_back(e - b);
    }
  } else {
    rb.push_back(g->row_begin);
    rn.push_back(g->n_rows);
  }
}

// Collectives run with a real NCCL communicator of > 1 rank -- or, with
// KDB_NCCL_FORCE=1 (tests), on a 1-rank NCCL communicator too, so one GPU runs
// the multi-rank host logic (exact per-round counts, agreed branches) through
// real NCCL calls.
bool multi_rank(const kdb_comm* comm) {
  if (!comm || comm->kind != 1) return false;
  if (comm->nranks > 1) return true;
  const char* f = getenv("KDB_NCCL_FORCE");
  return f && atoi(f) != 0;
}

kdb_status allreduce_min_u64(kdb_comm* comm, uint64_t* p, int64_t n, cudaStream_t st) {
  if (!multi_rank(comm) || n <= 0) return KDB_OK;
  return nccl_check(g_nccl.AllReduce(p, p, (size_t)n, ncclUint64, ncclMin, comm->nccl, st), "ncclAllReduce(u64,min)");
}
kdb_status allreduce_min_u32(kdb_comm* comm, uint32_t* p, int64_t n, cudaStream_t st) {
  if (!multi_rank(comm) || n <= 0) return KDB_OK;
  return nccl_check(g_nccl.AllReduce(p, p, (size_t)n, ncclUint32, ncclMin, comm->nccl, st), "ncclAllReduce(u32,min)");
}

kdb_status allreduce_max_u32(kdb_comm* comm, uint32_t* p, int64_t n, cudaStream_t st) {
  if (!multi_rank(comm) || n <= 0) return KDB_OK;
  return nccl_check(g_nccl.AllReduce(p, p, (size_t)n, ncclUint32, ncclMax, comm->nccl, st), "ncclAllReduce(u32,max)");
}

int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

// One kdb_mst call: the workspace layout plus the phase bookkeeping.
struct Mst {
  Layout L;
  const kdb_graph* g = nullptr;
  kdb_comm* comm = nullptr;
  cudaStream_t st = nullptr;
  int64_t N = 0;
  int32_t k = 0;   // candidate columns: edge_cols (kdb.h), else k_max
  int32_t ld = 0;  // row stride k_max
  const uint32_t* bits = nullptr;
  int32_t* comp = nullptr;
  bool general = false;
  int64_t C = 0;         // components after the rows phase (light components under the filter)
  int64_t C_heavy = -1;  // components after the heavy phase (-1: no heavy phase ran)
  // bytes per rank carried by the MIN all-reduces over component arrays (issued
  // with a communicator; counted either way): rows phase, heavy / cut phase
  double payload_rows = 0, payload_heavy = 0;
  int rounds = 0, stalls = 0, heavy_rounds = 0;
  double t_init = 0, t_inlist = 0, t_min_edges = 0, t_contract = 0, t_filter = 0, t_heavy = 0;
  unsigned long long entries = 0, survivors = 0, exceptions = 0, slow_entries = 0;
  float tau = 0.f;
  int fallback = 0;
  cudaEvent_t ev[4];
};

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// Light threshold: the median of column m0-1 over sampled local rows, made
// global with an all-reduce MIN (all ranks must filter with the same tau).
kdb_status pick_tau(Mst& m, int m0, float* tau_out) {
  const kdb_graph* g = m.g;
  Layout& L = m.L;
  const int64_t n = g->n_rows;
  uint32_t tb = kInfBits;
  if (n > 0) {
    const int64_t S = std::min<int64_t>(n, kTauSamples);
    const int64_t stride = n / S;
    LAUNCH(k_sample_col, grid_for(S), kThreads, m.st, g->dist, n, m.ld, m0 - 1, stride, S, L.tau_sample);
    KDB_CUDA(cudaGetLastError());
    std::vector<float> h(S);
    KDB_CUDA(cudaMemcpyAsync(h.data(), L.tau_sample, S * sizeof(float), cudaMemcpyDeviceToHost, m.st));
    KDB_CUDA(cudaStreamSynchronize(m.st));
    std::nth_element(h.begin(), h.begin() + S / 2, h.end());
    float t = h[S / 2];
    if (!(t >= 0.f)) t = __builtin_inff();  // NaN guard
    memcpy(&tb, &t, 4);
    if (tb == 0x80000000u) tb = 0u;
  }
  if (multi_rank(m.comm)) {
    uint32_t* d = reinterpret_cast<uint32_t*>(L.tau_sample);
    KDB_CUDA(cudaMemcpyAsync(d, &tb, 4, cudaMemcpyHostToDevice, m.st));
    KDB_TRY(allreduce_min_u32(m.comm, d, 1, m.st));
    KDB_CUDA(cudaMemcpyAsync(&tb, d, 4, cudaMemcpyDeviceToHost, m.st));
    KDB_CUDA(cudaStreamSynchronize(m.st));
  }
  memcpy(tau_out, &tb, 4);
  return KDB_OK;
}

// a2-a8: rows-Boruvka over the candidate entries with w <= eps_run (from
// singletons).  Leaves comp[] = dense component ids (0..C-1), L.cmin = minimum
// core id per component, m.C.  Resets the MSF counter.
kdb_status rows_phase(Mst& m, float eps_run) {
  Layout& L = m.L;
  kdb_comm* comm = m.comm;
  cudaStream_t st = m.st;
  const int64_t N = m.N;
  const int32_t k = m.k;    // candidate columns (edge_cols)
  const int32_t ld = m.ld;  // row stride
  const uint32_t* core_bits = m.bits;
  int32_t* comp = m.comp;
  const bool general = m.general;
  const bool vec = (ld % 4) == 0;
  cudaEvent_t* ev = m.ev;
  KDB_CUDA(cudaEventRecord(ev[0], st));

  // ---- a2: dense component ids -------------------------------------------------
  const int64_t nwords = (N + 31) / 32;
  uint32_t* popc = reinterpret_cast<uint32_t*>(L.flag);  // scratch, nwords + 1 <= N + 1
  KDB_CUDA(cudaMemsetAsync(popc + nwords, 0, sizeof(uint32_t), st));
  KDB_CUDA(cudaMemsetAsync(L.ctr, 0, sizeof(RoundCounters), st));
  LAUNCH(k_popc_words, grid_for(nwords), kThreads, st, core_bits, nwords, popc);
  KDB_CUDA(cudaGetLastError());
  size_t cb = L.cub_bytes;
  { LaunchScope ls_("cub::DeviceScan", st, false); KDB_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb, popc, L.woff, (int)(nwords + 1), st)); }
  uint32_t C32 = 0;  // woff[nwords] = number of core points
  KDB_CUDA(cudaMemcpyAsync(&C32, L.woff + nwords, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  KDB_CUDA(cudaStreamSynchronize(st));
  int64_t C = C32;
  L.all_core = (C == N) ? 1 : 0;  // then the dense id of a vertex is the vertex itself
  LAUNCH(k_init_comp, grid_for(N), kThreads, st, core_bits, L.woff, N, comp, L.cmin);
  LAUNCH(k_fill_comp_arrays, grid_for(C), kThreads, st, C, L.Kc, L.Bc, general ? nullptr : L.kmin);
  for (size_t r = 1; r < L.ranks.size(); ++r)
    LAUNCH(k_fill_comp_arrays, grid_for(C), kThreads, st, C, L.ranks[r].Kc, L.ranks[r].Bc, nullptr);
  KDB_CUDA(cudaGetLastError());
  const bool use_compact = env_int("KDB_COMPACT", 1) != 0;
  const int gw = env_int("KDB_GW", 4);  // component-gather width of the later light rounds (scan_ell)
  const bool sparse_ids = env_int("KDB_SPARSE", 1) != 0;  // keep root ids once few components remain
  // exact mode: round 1 (singleton components) is fused into the ELL pass; a
  // single rank also packs (K, B, kmin) per component for the round-1 hook
  const bool fuse1 = !general && use_compact && env_int("KDB_FUSE1", 1) != 0;
  const bool packed1 = fuse1 && L.ranks.size() == 1 && !(multi_rank(comm)) &&
                       env_int("KDB_PACK1", 1) != 0;
  if (!general)  // hook targets of round 1 (written by the round-1 offers)
    for (auto& R : L.ranks) LAUNCH(k_fill_i32, grid_for(C), kThreads, st, R.tgt, C, INT32_MAX);
  for (auto& R : L.ranks) {
    KDB_CUDA(cudaMemsetAsync(R.ctr, 0, sizeof(RoundCounters), st));
    R.compact = false;
    if (R.n_rows > 0 && use_compact) {
      R.compact = true;
      // 32-byte sector loads need 32-B aligned arrays, ld % 8 in {0, 4} and rows
      // long enough for the third sector (ld >= 20)
      const bool a32 = vec && ld >= 20 && !(((uintptr_t)R.nbr | (uintptr_t)R.dist) & 31u);
#define KDB_ELL_LAUNCH(V, A)                                                                                    \
  LAUNCH((k_light_ell<V, A>), grid_for(R.n_rows), kThreads, st, R.nbr, R.dist, R.n_rows, ld, k, eps_run, R.row_begin, \
         comp, general ? nullptr : L.kmin, R.LE, R.act[0], &R.ctr->na[0], &R.ctr->grab, fuse1 ? 1 : 0,         \
         L.all_core, N, R.Kc, R.Bc, R.tgt, packed1 ? L.rec1 : nullptr)
      if (a32) KDB_ELL_LAUNCH(true, true);
      else if (vec) KDB_ELL_LAUNCH(true, false);
      else KDB_ELL_LAUNCH(false, false);
#undef KDB_ELL_LAUNCH
    }
    if (R.n_rows > 0 && !R.compact)
      LAUNCH(k_init_rows, grid_for(R.n_rows), kThreads, st, R.dist, R.n_rows, ld, k, eps_run, R.row_begin, comp,
             general ? nullptr : L.kmin, R.act[0], &R.ctr->na[0]);
    KDB_CUDA(cudaGetLastError());
  }
  if (!general) KDB_TRY(allreduce_min_u32(comm, L.kmin, C, st));
  if (!general) m.payload_rows += 4.0 * C;
  KDB_CUDA(cudaEventRecord(ev[1], st));
  // ---- general mode: in-edge lists --------------------------------------------
  if (general) {
    for (auto& R : L.ranks) {
      // counts -> scan -> offsets; e_key (N+1 u64) is scratch for counts and cursors
      unsigned long long* cursor = reinterpret_cast<unsigned long long*>(L.e_key);
      KDB_CUDA(cudaMemsetAsync(cursor, 0, (N + 1) * sizeof(unsigned long long), st));
      if (R.n_rows > 0)
        LAUNCH(k_in_count, grid_for(R.n_rows), kThreads, st, R.nbr, R.dist, R.n_rows, ld, k, eps_run, R.row_begin, N,
               core_bits, cursor);
      cb = L.cub_bytes;
      { LaunchScope ls_("cub::DeviceScan", st, false); KDB_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb, cursor, R.in_off, (int)(N + 1), st)); }
      KDB_CUDA(cudaMemcpyAsync(cursor, R.in_off, (N + 1) * sizeof(unsigned long long),
                               cudaMemcpyDeviceToDevice, st));
      if (R.n_rows > 0)
        LAUNCH(k_in_fill, grid_for(R.n_rows), kThreads, st, R.nbr, R.dist, R.n_rows, ld, k, eps_run, R.row_begin, N,
               core_bits, cursor, R.in_src, R.in_w);
      LAUNCH(k_in_finish, grid_for(N), kThreads, st, R.in_off, N, R.in_len, R.in_act[0], &R.ctr->ni[0]);
      KDB_CUDA(cudaGetLastError());
    }
  }
  for (auto& R : L.ranks) {
    RoundCounters hc;
    KDB_CUDA(cudaMemcpyAsync(&hc, R.ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    R.n_act = hc.na[0];
    R.n_in_act = hc.ni[0];
  }
  KDB_CUDA(cudaEventRecord(ev[2], st));
  KDB_CUDA(cudaEventSynchronize(ev[2]));
  m.t_init += elapsed(ev[0], ev[1]);
  m.t_inlist += elapsed(ev[1], ev[2]);

  // ---- Boruvka rounds -------------------------------------------------------------
  // Pipelined: every kernel reads its counts (components, list sizes) from the
  // device; grids are sized by host upper bounds one round stale, so the host
  // enqueues round r+1 before it has looked at round r and checks round r-1's
  // counters (termination, violations, stalls) from pinned memory meanwhile.
  // A round launched after the last productive one finds nothing and changes
  // nothing.  With a real NCCL communicator the collectives need exact host
  // counts: the loop then waits for each round's counters (sync_each).
  bool any_compact = false;
  for (auto& R : L.ranks) any_compact |= R.compact;
  const bool fused = fuse1 && any_compact;
  const bool sync_each = multi_rank(comm);
  int cur = fused ? 1 : 0;  // fused round 1: its OUTPUT list is act[0] already
  int par = 0;              // component count ping-pong: Cs[par] current
  {
    long long c0 = C;
    KDB_CUDA(cudaMemcpyAsync(&L.ctr->Cs[0], &c0, sizeof(c0), cudaMemcpyHostToDevice, st));
  }
  const size_t nr = L.ranks.size();
  // pinned slots for the round counters: [0] global, [1 + r] rank r
  constexpr int kSlots = 4;
  // (a per-thread pinned buffer, grown on demand: cudaMallocHost per call is slow)
  static thread_local RoundCounters* slots = nullptr;
  static thread_local size_t slots_cap = 0;
  if (slots_cap < kSlots * (1 + nr)) {
    if (slots) cudaFreeHost(slots);
    slots = nullptr;
    slots_cap = 0;
    KDB_CUDA(cudaMallocHost(&slots, kSlots * (1 + nr) * sizeof(RoundCounters)));
    slots_cap = kSlots * (1 + nr);
  }
  std::vector<cudaEvent_t> ev_slot(kSlots), ev_rnd;
  for (auto& e : ev_slot) KDB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  struct EvVecGuard {
    std::vector<cudaEvent_t>* a;
    std::vector<cudaEvent_t>* b;
    ~EvVecGuard() {
      for (auto e : *a) cudaEventDestroy(e);
      for (auto e : *b) cudaEventDestroy(e);
    }
  } evg{&ev_slot, &ev_rnd};
  int64_t C_ub = C;  // upper bound of the current component count
  std::vector<uint32_t> na_ub(nr), ni_ub(nr);
  for (size_t r = 0; r < nr; ++r) {
    na_ub[r] = L.ranks[r].n_act;
    ni_ub[r] = L.ranks[r].n_in_act;
  }
  int rounds = 0, stalls = 0;
  const uint32_t* kmin_cert = general ? nullptr : L.kmin;
  auto slot_of = [&](int rr) { return slots + (size_t)(rr % kSlots) * (1 + nr); };

  // contraction a6 on the device counts; C_bound >= the true count
  auto contract = [&](int64_t C_bound) -> kdb_status {
    const int64_t* Cd = (const int64_t*)&L.ctr->Cs[par];
    int64_t* Cn = (int64_t*)&L.ctr->Cs[par ^ 1];
    LAUNCH(k_jump, grid_for(C_bound), kThreads, st, C_bound, L.parent, L.rootof, L.ctr, Cd);
    // sparse ids once few components remain: a component keeps its root's id
    // (no dense renumbering; the id range stays C_bound), so the relabel only
    // rewrites the vertices of merged components
    const bool sparse = sparse_ids && C_bound <= N / 64;
    if (!sparse) {
      LAUNCH(k_root_flags, grid_for(C_bound), kThreads, st, C_bound, L.rootof, L.flag, Cd);
      size_t cb2 = L.cub_bytes;
      { LaunchScope ls_("cub::DeviceScan", st, false); KDB_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb2, L.flag, L.newid, (int)std::max<int64_t>(C_bound, 1), st)); }
      LAUNCH(k_count_roots, 1, 1, st, Cd, L.newid, L.flag, Cn);
    } else {
      KDB_CUDA(cudaMemcpyAsync(Cn, Cd, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    }
    LAUNCH(k_fill_i32, grid_for(C_bound), kThreads, st, L.cmin2, C_bound, INT32_MAX, (const int64_t*)Cn);
    if (!general)
      LAUNCH(k_fill_i32, grid_for(C_bound), kThreads, st, (int32_t*)L.kmin2, C_bound, (int32_t)kInfBits,
             (const int64_t*)Cn);
    // map[c] = new dense id of c's tree (reuses `parent`, no longer needed)
    LAUNCH(k_merge, grid_for(C_bound), kThreads, st, C_bound, L.rootof, sparse ? (const int32_t*)nullptr : L.newid,
           L.cmin, general ? nullptr : L.kmin, L.cmin2, L.kmin2, L.parent, Cd);
    LAUNCH(k_relabel, grid_for(N / 8 + 1), kThreads, st, N, comp, L.parent, (const int32_t*)nullptr);
    LAUNCH(k_fill_comp_arrays, grid_for(C_bound), kThreads, st, C_bound, L.Kc, L.Bc, nullptr, (const int64_t*)Cn);
    for (size_t r = 1; r < nr; ++r)
      LAUNCH(k_fill_comp_arrays, grid_for(C_bound), kThreads, st, C_bound, L.ranks[r].Kc, L.ranks[r].Bc, nullptr,
             (const int64_t*)Cn);
    KDB_CUDA(cudaGetLastError());
    std::swap(L.cmin, L.cmin2);
    std::swap(L.kmin, L.kmin2);
    kmin_cert = general ? nullptr : L.kmin;
    par ^= 1;
    return KDB_OK;
  };
  // snapshot of the counters after the current round into a pinned slot
  auto snapshot = [&](int rr) -> kdb_status {
    RoundCounters* sl = slot_of(rr);
    KDB_CUDA(cudaMemcpyAsync(sl, L.ctr, sizeof(RoundCounters), cudaMemcpyDeviceToHost, st));
    for (size_t r = 0; r < nr; ++r)
      KDB_CUDA(cudaMemcpyAsync(sl + 1 + r, L.ranks[r].ctr, sizeof(RoundCounters), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaEventRecord(ev_slot[rr % kSlots], st));
    return KDB_OK;
  };

  int last_checked = 0;
  bool finished = false;
  while (!finished) {
    ++rounds;
    const bool direct = rounds == 1 && !general;
    const int64_t* Cd = (const int64_t*)&L.ctr->Cs[par];
    cudaEvent_t e0;
    KDB_CUDA(cudaEventCreate(&e0));
    ev_rnd.push_back(e0);
    KDB_CUDA(cudaEventRecord(e0, st));
    // offers read the current key before their atomicMin once many rows offer
    // to each component (same-address atomics serialise; early rounds have
    // about one row per component and only pay the extra read)
    int precheck = 0;
    {
      uint64_t live = 0;
      for (size_t r = 0; r < nr; ++r) live += na_ub[r];
      const int pc = env_int("KDB_PRECHECK", -1);
      precheck = pc >= 0 ? pc : (live > 8 * (uint64_t)std::max<int64_t>(C_ub, 1) ? 1 : 0);
    }
    // a3: offers (rows, then in-lists), per rank, into that rank's Kc partial
    for (size_t r = 0; r < nr; ++r) {
      RankState& R = L.ranks[r];
      if (direct && fused && R.compact) continue;  // done by the ELL pass
      KDB_CUDA(cudaMemsetAsync(&R.ctr->na[cur ^ 1], 0, sizeof(uint32_t), st));
      KDB_CUDA(cudaMemsetAsync(&R.ctr->ni[cur ^ 1], 0, sizeof(uint32_t), st));
      KDB_CUDA(cudaMemsetAsync(&R.ctr->n_off, 0, sizeof(uint32_t), st));
      KDB_CUDA(cudaMemsetAsync(&R.ctr->grab, 0, sizeof(uint32_t), st));
      const uint32_t* nin = &R.ctr->na[cur];
      uint32_t* nout = &R.ctr->na[cur ^ 1];
      if (na_ub[r] && R.compact) {
        if (direct)
          LAUNCH(k_light_first, grid_for(na_ub[r]), kThreads, st, R.LE, R.nbr, R.dist, ld, k, eps_run, R.row_begin, N,
                 comp, L.all_core, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, R.Kc, R.Bc, R.tgt,
                 &L.ctr->entries, nin);
        else
        {
#define KDB_LR_LAUNCH(GW)                                                                                       \
  LAUNCH(k_light_round<GW>, grid_for(na_ub[r]), kThreads, st, R.LE, R.nbr, R.dist, ld, k, eps_run, R.row_begin, N, \
         comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, R.offers, (unsigned long long*)R.Kc,      \
         &L.ctr->entries, nin, precheck)
          if (gw == 1) KDB_LR_LAUNCH(1);
          else if (gw == 2) KDB_LR_LAUNCH(2);
          else KDB_LR_LAUNCH(4);
#undef KDB_LR_LAUNCH
        }
      } else if (na_ub[r]) {
        if (direct) {
          if (vec)
            LAUNCH(k_offer_first<true>, grid_for(na_ub[r]), kThreads, st, R.nbr, R.dist, ld, k, eps_run, R.row_begin, N,
                   comp, L.all_core, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, R.Kc, R.Bc, R.tgt,
                   &L.ctr->entries, nin);
          else
            LAUNCH(k_offer_first<false>, grid_for(na_ub[r]), kThreads, st, R.nbr, R.dist, ld, k, eps_run, R.row_begin,
                   N, comp, L.all_core, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, R.Kc, R.Bc, R.tgt,
                   &L.ctr->entries, nin);
        } else {
          if (vec)
            LAUNCH(k_offer_round<true>, grid_for(na_ub[r]), kThreads, st, R.nbr, R.dist, ld, k, eps_run, R.row_begin, N,
                   comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, R.offers, (unsigned long long*)R.Kc,
                   &L.ctr->entries, nin, precheck);
          else
            LAUNCH(k_offer_round<false>, grid_for(na_ub[r]), kThreads, st, R.nbr, R.dist, ld, k, eps_run, R.row_begin,
                   N, comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, R.offers, (unsigned long long*)R.Kc,
                   &L.ctr->entries, nin, precheck);
        }
      }
      if (general && ni_ub[r])
        LAUNCH(k_offer_in, grid_for(ni_ub[r]), kThreads, st, R.in_off, R.in_len, R.in_src, R.in_w, comp,
               R.in_act[cur], ni_ub[r], R.in_act[cur ^ 1], &R.ctr->ni[cur ^ 1], R.offers + R.off_cap_rows,
               &R.ctr->n_off, (unsigned long long*)R.Kc, &R.ctr->ni[cur]);
      KDB_CUDA(cudaGetLastError());
    }
    // exchange: sim -> min over virtual ranks; nccl -> allreduce
    for (size_t r = 1; r < nr; ++r)
      LAUNCH(k_min_into_u64, grid_for(C_ub), kThreads, st, L.Kc, L.ranks[r].Kc, C_ub, Cd);
    KDB_TRY(allreduce_min_u64(comm, L.Kc, C_ub, st));
    m.payload_rows += 8.0 * C_ub;
    // a4: ties (the direct round already wrote Bc and the targets)
    if (!direct) {
      for (size_t r = 0; r < nr; ++r) {
        RankState& R = L.ranks[r];
        if (na_ub[r]) LAUNCH(k_tie, grid_for(na_ub[r]), kThreads, st, R.offers, &R.ctr->na[cur ^ 1], L.Kc, R.Bc);
        if (general && ni_ub[r])
          LAUNCH(k_tie, grid_for(ni_ub[r]), kThreads, st, R.offers + R.off_cap_rows, &R.ctr->n_off, L.Kc, R.Bc);
        KDB_CUDA(cudaGetLastError());
      }
    }
    for (size_t r = 1; r < nr; ++r)
      LAUNCH(k_min_into_u32, grid_for(C_ub), kThreads, st, L.Bc, L.ranks[r].Bc, C_ub, Cd);
    KDB_TRY(allreduce_min_u32(comm, L.Bc, C_ub, st));
    m.payload_rows += 4.0 * C_ub;
    if (direct) {
      for (size_t r = 1; r < nr; ++r)
        LAUNCH(k_min_into_u32, grid_for(C_ub), kThreads, st, (uint32_t*)L.tgt, (const uint32_t*)L.ranks[r].tgt, C_ub,
               Cd);
      KDB_TRY(allreduce_min_u32(comm, (uint32_t*)L.tgt, C_ub, st));  // non-owners hold INT32_MAX
      m.payload_rows += 4.0 * C_ub;
    }
    // a5: hook + emit
    KDB_CUDA(cudaMemsetAsync(&L.ctr->hooks, 0, 4 * sizeof(uint32_t), st));
    if (direct && packed1)
      LAUNCH(k_hook<true>, grid_for(C_ub), kThreads, st, C_ub, L.Kc, L.Bc, L.tgt, kmin_cert, comp, L.parent, L.e_key,
             L.e_w, N, L.ctr, Cd, L.rec1);
    else
      LAUNCH(k_hook<false>, grid_for(C_ub), kThreads, st, C_ub, L.Kc, L.Bc, direct ? L.tgt : nullptr, kmin_cert,
             comp, L.parent, L.e_key, L.e_w, N, L.ctr, Cd, (const int4*)nullptr);
    KDB_CUDA(cudaGetLastError());
    // a6: contract (no hooks => identity)
    KDB_TRY(contract(C_ub));
    cur ^= 1;
    KDB_TRY(snapshot(rounds));
    // check the previous round (or this one when every round must be exact)
    const int check = sync_each ? rounds : rounds - 1;
    if (check < 1 || check <= last_checked) continue;
    KDB_CUDA(cudaEventSynchronize(ev_slot[check % kSlots]));
    last_checked = check;
    const RoundCounters g = slot_of(check)[0];
    if (g_trace)
      fprintf(stderr, "[kdb] round %d eps=%.6g C->%lld offered=%u hooks=%u live=%u\n", check, (double)eps_run,
              (long long)g.Cs[(check & 1) ? 1 : 0], g.offered, g.hooks, slot_of(check)[1].na[check & 1]);
    if (g.violation == 2u) return set_err(KDB_EINTERNAL, "pointer jumping did not converge (hook cycle)");
    if (g.violation) return set_err(KDB_EINVAL, "graph violates the KDB_GRAPH_EXACT promise (a component's "
                                    "minimum missed an incident edge)");
    if (g.offered == 0) break;  // a8: no component has a leaving edge
    // upper bounds for the next launch: the counts after round `check`
    {
      // after round `check` the current parity was flipped `rounds - check` more times
      const int par_after = (par ^ ((rounds - check) & 1));
      C_ub = g.Cs[par_after];
      const int cur_after = (cur ^ ((rounds - check) & 1));
      for (size_t r = 0; r < nr; ++r) {
        na_ub[r] = slot_of(check)[1 + r].na[cur_after];
        ni_ub[r] = slot_of(check)[1 + r].ni[cur_after];
      }
    }
    if (g.hooks == 0) {
      // every offering component abstained (exact-mode certificate).  Drain,
      // then one edge-centric sweep round gives every component its exact
      // minimum (both endpoints see every entry) -- on exact counts.
      ++stalls;
      KDB_CUDA(cudaStreamSynchronize(st));
      RoundCounters gg;
      KDB_CUDA(cudaMemcpy(&gg, L.ctr, sizeof(gg), cudaMemcpyDeviceToHost));
      if (gg.violation) return set_err(KDB_EINVAL, "graph violates the KDB_GRAPH_EXACT promise (a component's "
                                       "minimum missed an incident edge)");
      const int64_t Cx = gg.Cs[par];
      std::vector<uint32_t> na_x(nr);
      for (size_t r = 0; r < nr; ++r) {
        RoundCounters rc;
        KDB_CUDA(cudaMemcpy(&rc, L.ranks[r].ctr, sizeof(rc), cudaMemcpyDeviceToHost));
        na_x[r] = rc.na[cur];
      }
      LAUNCH(k_fill_comp_arrays, grid_for(Cx), kThreads, st, Cx, L.Kc, L.Bc, nullptr);
      for (size_t r = 1; r < nr; ++r)
        LAUNCH(k_fill_comp_arrays, grid_for(Cx), kThreads, st, Cx, L.ranks[r].Kc, L.ranks[r].Bc, nullptr);
      for (size_t r = 0; r < nr; ++r)
        if (na_x[r])
          LAUNCH(k_sweep, grid_for(na_x[r]), kThreads, st, L.ranks[r].nbr, L.ranks[r].dist, ld, k, eps_run,
                 L.ranks[r].row_begin, N, comp, L.ranks[r].act[cur], na_x[r], (unsigned long long*)L.ranks[r].Kc,
                 L.ranks[r].Bc, 0);
      for (size_t r = 1; r < nr; ++r)
        LAUNCH(k_min_into_u64, grid_for(Cx), kThreads, st, L.Kc, L.ranks[r].Kc, Cx);
      KDB_TRY(allreduce_min_u64(comm, L.Kc, Cx, st));
      m.payload_rows += 8.0 * Cx;
      for (size_t r = 0; r < nr; ++r)
        if (na_x[r])
          LAUNCH(k_sweep, grid_for(na_x[r]), kThreads, st, L.ranks[r].nbr, L.ranks[r].dist, ld, k, eps_run,
                 L.ranks[r].row_begin, N, comp, L.ranks[r].act[cur], na_x[r], (unsigned long long*)L.Kc,
                 L.ranks[r].Bc, 1);
      for (size_t r = 1; r < nr; ++r)
        LAUNCH(k_min_into_u32, grid_for(Cx), kThreads, st, L.Bc, L.ranks[r].Bc, Cx);
      KDB_TRY(allreduce_min_u32(comm, L.Bc, Cx, st));
      m.payload_rows += 4.0 * Cx;
      KDB_CUDA(cudaMemsetAsync(&L.ctr->hooks, 0, 4 * sizeof(uint32_t), st));
      LAUNCH(k_hook<false>, grid_for(Cx), kThreads, st, Cx, L.Kc, L.Bc, nullptr, nullptr, comp, L.parent, L.e_key,
             L.e_w, N, L.ctr, (const int64_t*)nullptr, (const int4*)nullptr);
      KDB_CUDA(cudaGetLastError());
      KDB_CUDA(cudaMemcpyAsync(&gg, L.ctr, sizeof(gg), cudaMemcpyDeviceToHost, st));
      KDB_CUDA(cudaStreamSynchronize(st));
      if (gg.hooks == 0) return set_err(KDB_EINTERNAL, "sweep round made no progress");
      KDB_TRY(contract(Cx));
      C_ub = Cx;
      for (size_t r = 0; r < nr; ++r) na_ub[r] = na_x[r];
      ++rounds;
      KDB_TRY(snapshot(rounds));
      last_checked = rounds;  // the sweep round was exact; the next check is the next round
    }
  }
  KDB_CUDA(cudaStreamSynchronize(st));
  if (!ev_rnd.empty()) {
    KDB_CUDA(cudaEventRecord(ev[2], st));
    KDB_CUDA(cudaEventSynchronize(ev[2]));
    m.t_min_edges += elapsed(ev_rnd.front(), ev[2]);  // rounds are pipelined: one span
  }
  {
    RoundCounters gg;
    KDB_CUDA(cudaMemcpy(&gg, L.ctr, sizeof(gg), cudaMemcpyDeviceToHost));
    C = gg.Cs[par];
  }
  RoundCounters hc;
  KDB_CUDA(cudaMemcpyAsync(&hc, L.ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
  KDB_CUDA(cudaStreamSynchronize(st));
  m.entries += hc.entries;
  m.rounds += rounds;
  m.stalls += stalls;
  m.C = C;
  return KDB_OK;
}

// Filter: every rank streams its rows once and keeps the heavy candidate
// entries (tau < w <= eps) whose endpoints lie in different light components.
kdb_status filter_phase(Mst& m, float eps, bool* overflow) {
  Layout& L = m.L;
  cudaStream_t st = m.st;
  KDB_CUDA(cudaEventRecord(m.ev[0], st));
  // KDB_SURVCAP (tests): a smaller survivor capacity, to exercise the fallback
  const int64_t cap_env = env_int("KDB_SURVCAP", -1);
  // fast-path tables (identical on every rank: comp is replicated)
  int shift = 0;
  while (((m.N + ((int64_t)1 << shift) - 1) >> shift) > kDomMax) ++shift;
  const int64_t nblk = (m.N + ((int64_t)1 << shift) - 1) >> shift;
  bool fast = env_int("KDB_FASTFILTER", 1) != 0;
  unsigned long long fc[2] = {0, 0};
  int2* rng = reinterpret_cast<int2*>(L.Kc);  // C_L entries; Kc is refilled by the heavy phase
  KDB_CUDA(cudaMemsetAsync(L.fcount, 0, 2 * sizeof(unsigned long long), st));
  if (fast) {
    const int64_t C = m.C;
    KDB_CUDA(cudaMemsetAsync(L.bloom, 0, kBloomBits / 8, st));
    LAUNCH(k_dom, grid_for(nblk * 32), kThreads, st, m.comp, m.N, shift, nblk, L.dom);
    LAUNCH(k_bloom_build, grid_for(m.N), kThreads, st, m.comp, m.N, shift, L.dom, L.bloom,
           reinterpret_cast<uint32_t*>(L.fcount));
    LAUNCH(k_fill_i32, grid_for(C), kThreads, st, L.parent, C, INT32_MAX);
    LAUNCH(k_fill_i32, grid_for(C), kThreads, st, L.rootof, C, -1);
    LAUNCH(k_fill_i32, grid_for(C), kThreads, st, L.newid, C, 0);
    LAUNCH(k_rng_acc, grid_for(nblk), kThreads, st, L.dom, nblk, L.parent, L.rootof, L.newid);
    LAUNCH(k_rng_fin, grid_for(C), kThreads, st, C, m.N, shift, L.parent, L.rootof, L.newid, rng);
    KDB_CUDA(cudaGetLastError());
    KDB_CUDA(cudaMemcpyAsync(fc, L.fcount, sizeof(fc), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    fc[0] &= 0xffffffffull;  // block_count wrote the low 32-bit word
    m.exceptions = fc[0];
    // a saturated filter would send almost every entry down the slow path
    if (fc[0] > (unsigned long long)kBloomBits / 4) fast = false;
  }
  for (auto& R : L.ranks) {
    KDB_CUDA(cudaMemsetAsync(R.n_hs_dev, 0, 2 * sizeof(uint32_t), st));
    if (cap_env >= 0) R.hs_cap = (uint32_t)std::min<int64_t>(R.hs_cap, cap_env);
    if (R.n_rows == 0) continue;
    const int vec = (m.ld % 4) == 0 ? 4 : 1;
    const bool cols = m.k < m.ld;  // edge_cols < row stride
    FastDiv fd;  // entry (COLS: chunk) index within a tile -> row within the tile
    fd.d = cols ? (uint64_t)((m.k + vec - 1) / vec) : (uint64_t)m.ld;
    fd.M = fd.d > 1 ? (~0ull / fd.d) + 1 : 0;
    fd.m32 = fd.d > 1 ? (uint32_t)((0xffffffffull / fd.d) + 1) : 0;
    fd.small = (fd.d > 1 && fd.d < 2048) ? 1u : 0u;
    const int64_t ntiles = (R.n_rows + kFilterThreads - 1) / kFilterThreads;
    const int grid = (int)std::min<int64_t>(ntiles, 1 << 30);
#define KDB_FILTER_LAUNCH(V, F, CO)                                                                              \
  LAUNCH_DYN((k_filter<V, F, CO>), grid, kFilterThreads, kFilterSmem, st, R.nbr, R.dist, R.n_rows, m.ld, m.k,      \
             m.tau, eps, R.row_begin, m.N, m.comp, rng, L.bloom, fd, R.hs[0], R.hs_cap, R.n_hs_dev, L.fcount + 1)
    if (cols) {
      if (vec == 4 && fast) KDB_FILTER_LAUNCH(4, true, true);
      else if (vec == 4) KDB_FILTER_LAUNCH(4, false, true);
      else if (fast) KDB_FILTER_LAUNCH(1, true, true);
      else KDB_FILTER_LAUNCH(1, false, true);
    } else {
      if (vec == 4 && fast) KDB_FILTER_LAUNCH(4, true, false);
      else if (vec == 4) KDB_FILTER_LAUNCH(4, false, false);
      else if (fast) KDB_FILTER_LAUNCH(1, true, false);
      else KDB_FILTER_LAUNCH(1, false, false);
    }
#undef KDB_FILTER_LAUNCH
    KDB_CUDA(cudaGetLastError());
  }
  uint32_t over = 0;
  unsigned long long tot = 0;
  for (auto& R : L.ranks) {
    uint32_t n = 0;
    KDB_CUDA(cudaMemcpyAsync(&n, R.n_hs_dev, 4, cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    R.n_hs = n;
    tot += n;
    if (n > R.hs_cap) over = 1;
  }
  if (multi_rank(m.comm)) {  // every rank must take the same branch
    uint32_t* d = L.ranks[0].n_hs_dev + 1;
    KDB_CUDA(cudaMemcpyAsync(d, &over, 4, cudaMemcpyHostToDevice, st));
    KDB_TRY(allreduce_max_u32(m.comm, d, 1, st));
    KDB_CUDA(cudaMemcpyAsync(&over, d, 4, cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
  }
  KDB_CUDA(cudaMemcpyAsync(&fc[1], L.fcount + 1, 8, cudaMemcpyDeviceToHost, st));
  KDB_CUDA(cudaStreamSynchronize(st));
  m.slow_entries = fc[1];
  KDB_CUDA(cudaEventRecord(m.ev[1], st));
  m.t_filter += elapsed(m.ev[0], m.ev[1]);
  m.survivors = tot;
  *overflow = over != 0;
  return KDB_OK;
}

// Heavy phase: edge-centric Boruvka over the survivors in light-component
// space.  hcomp maps light component -> current heavy component (replicated).
kdb_status heavy_phase(Mst& m) {
  Layout& L = m.L;
  cudaStream_t st = m.st;
  kdb_comm* comm = m.comm;
  const int64_t CL = m.C;
  int64_t C = CL;
  KDB_CUDA(cudaEventRecord(m.ev[0], st));
  LAUNCH(k_iota, grid_for(CL), kThreads, st, L.hcomp, CL);
  std::vector<int> cur(L.ranks.size(), 0);
  int rounds = 0;
  while (C > 1) {
    ++rounds;
    LAUNCH(k_fill_comp_arrays, grid_for(C), kThreads, st, C, L.Kc, L.Bc, nullptr);
    for (size_t r = 1; r < L.ranks.size(); ++r)
      LAUNCH(k_fill_comp_arrays, grid_for(C), kThreads, st, C, L.ranks[r].Kc, L.ranks[r].Bc, nullptr);
    for (size_t r = 0; r < L.ranks.size(); ++r) {
      RankState& R = L.ranks[r];
      if (R.n_hs == 0) continue;
      LAUNCH(k_hedge_offer, grid_for(R.n_hs), kThreads, st, R.hs[cur[r]], R.n_hs, L.hcomp,
             (unsigned long long*)R.Kc, R.hkeep);
      size_t cb = L.cub_bytes;
      { LaunchScope ls_("cub::DeviceSelect", st, false);
        KDB_CUDA(cub::DeviceSelect::Flagged(L.cub_tmp, cb, R.hs[cur[r]], R.hkeep, R.hs[cur[r] ^ 1],
                                            R.n_hs_dev + 1, (int)R.n_hs, st)); }
      cur[r] ^= 1;
      KDB_CUDA(cudaGetLastError());
    }
    for (auto& R : L.ranks) {
      if (R.n_hs == 0) continue;
      KDB_CUDA(cudaMemcpyAsync(&R.n_hs, R.n_hs_dev + 1, 4, cudaMemcpyDeviceToHost, st));
    }
    KDB_CUDA(cudaStreamSynchronize(st));
    for (size_t r = 1; r < L.ranks.size(); ++r)
      LAUNCH(k_min_into_u64, grid_for(C), kThreads, st, L.Kc, L.ranks[r].Kc, C);
    KDB_TRY(allreduce_min_u64(comm, L.Kc, C, st));
    m.payload_heavy += 8.0 * C;
    for (size_t r = 0; r < L.ranks.size(); ++r) {
      RankState& R = L.ranks[r];
      if (R.n_hs)
        LAUNCH(k_hedge_tie, grid_for(R.n_hs), kThreads, st, R.hs[cur[r]], R.n_hs, L.hcomp, L.Kc, R.Bc);
    }
    for (size_t r = 1; r < L.ranks.size(); ++r)
      LAUNCH(k_min_into_u32, grid_for(C), kThreads, st, L.Bc, L.ranks[r].Bc, C);
    KDB_TRY(allreduce_min_u32(comm, L.Bc, C, st));
    m.payload_heavy += 4.0 * C;
    KDB_CUDA(cudaMemsetAsync(&L.ctr->hooks, 0, 4 * sizeof(uint32_t), st));
    LAUNCH(k_hook_h, grid_for(C), kThreads, st, C, L.Kc, L.Bc, m.comp, L.hcomp, L.parent, L.e_key, L.e_w, m.N, L.ctr);
    KDB_CUDA(cudaGetLastError());
    RoundCounters hc;
    KDB_CUDA(cudaMemcpyAsync(&hc, L.ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    if (hc.offered == 0) break;
    if (hc.hooks == 0) return set_err(KDB_EINTERNAL, "heavy phase made no progress");
    LAUNCH(k_jump, grid_for(C), kThreads, st, C, L.parent, L.rootof, L.ctr);
    LAUNCH(k_root_flags, grid_for(C), kThreads, st, C, L.rootof, L.flag);
    size_t cb = L.cub_bytes;
    { LaunchScope ls_("cub::DeviceScan", st, false); KDB_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb, L.flag, L.newid, (int)C, st)); }
    uint32_t viol = 0;
    int32_t last[2];
    KDB_CUDA(cudaMemcpyAsync(&viol, &L.ctr->violation, 4, cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaMemcpyAsync(&last[0], L.newid + C - 1, 4, cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaMemcpyAsync(&last[1], L.flag + C - 1, 4, cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    if (viol) return set_err(KDB_EINTERNAL, "heavy-phase pointer jumping did not converge");
    const int64_t C2 = (int64_t)last[0] + last[1];
    LAUNCH(k_fill_i32, grid_for(C2), kThreads, st, L.cmin2, C2, INT32_MAX);
    LAUNCH(k_merge, grid_for(C), kThreads, st, C, L.rootof, L.newid, L.cmin, nullptr, L.cmin2, nullptr, L.parent);
    LAUNCH(k_relabel_h, grid_for(CL), kThreads, st, CL, L.hcomp, L.parent);
    KDB_CUDA(cudaGetLastError());
    std::swap(L.cmin, L.cmin2);
    C = C2;
  }
  KDB_CUDA(cudaEventRecord(m.ev[1], st));
  m.t_heavy += elapsed(m.ev[0], m.ev[1]);
  m.heavy_rounds = rounds;
  m.C_heavy = C;
  return KDB_OK;
}

}  // namespace

// ============================================================================
// C-ABI
// ============================================================================
extern "C" {

const char* kdb_status_string(kdb_status s) {
  switch (s) {
    case KDB_OK: return "KDB_OK";
    case KDB_EINVAL: return "KDB_EINVAL";
    case KDB_ENOMEM: return "KDB_ENOMEM";
    case KDB_ECUDA: return "KDB_ECUDA";
    case KDB_ENCCL: return "KDB_ENCCL";
    case KDB_EINTERNAL: return "KDB_EINTERNAL";
  }
  return "KDB_?";
}

const char* kdb_last_error(void) { return g_err.c_str(); }

int kdb_last_mst_stats(double* out, int cap) {
  int n = std::min(cap, 20);
  for (int i = 0; i < n; ++i) out[i] = g_stats[i];
  return n;
}

void kdb_profile_enable(int on) { g_prof.on = on != 0; }

void kdb_profile_reset(void) {
  g_prof.drain();
  g_prof.names.clear();
  g_prof.ms.clear();
  g_prof.cnt.clear();
  g_prof.launches = 0;
}

long long kdb_launch_count(void) { return g_prof.launches; }

int kdb_profile_read(char* names, size_t names_len, double* ms, long long* counts, int cap) {
  g_prof.drain();
  size_t off = 0;
  int n = 0;
  for (size_t i = 0; i < g_prof.names.size() && n < cap; ++i, ++n) {
    ms[n] = g_prof.ms[i];
    counts[n] = g_prof.cnt[i];
    const std::string& nm = g_prof.names[i];
    if (names && off + nm.size() + 1 < names_len) {
      memcpy(names + off, nm.c_str(), nm.size());
      off += nm.size();
      names[off++] = '\n';
      names[off] = 0;
    }
  }
  return n;
}

kdb_status kdb_nccl_unique_id(void* out) {
  if (!out) return set_err(KDB_EINVAL, "out is NULL");
  KDB_TRY(nccl_load());
  ncclUniqueId id;
  KDB_TRY(nccl_check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId"));
  memcpy(out, &id, sizeof(id));
  return KDB_OK;
}

kdb_status kdb_comm_create_nccl(kdb_comm** out, const void* uid, int rank, int nranks) {
  if (!out || !uid || nranks < 1 || rank < 0 || rank >= nranks)
    return set_err(KDB_EINVAL, "bad communicator arguments");
  KDB_TRY(nccl_load());
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  kdb_comm* c = new kdb_comm();
  c->kind = 1;
  c->rank = rank;
  c->nranks = nranks;
  kdb_status s = nccl_check(g_nccl.CommInitRank(&c->nccl, nranks, id, rank), "ncclCommInitRank");
  if (s != KDB_OK) {
    delete c;
    return s;
  }
  *out = c;
  return KDB_OK;
}

kdb_status kdb_comm_create_sim(kdb_comm** out, int nranks) {
  if (!out || nranks < 1 || nranks > 1024) return set_err(KDB_EINVAL, "bad sim rank count");
  kdb_comm* c = new kdb_comm();
  c->kind = 2;
  c->rank = 0;
  c->nranks = nranks;
  *out = c;
  return KDB_OK;
}

void kdb_comm_destroy(kdb_comm* c) {
  if (!c) return;
  if (c->kind == 1 && c->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy(c->nccl);
  delete c;
}

kdb_status kdb_core_mark(const kdb_graph* g, int32_t M, float eps, uint32_t* core_bits, kdb_comm* comm,
                         kdb_stream_t stream) {
  KDB_TRY(validate_graph(g));
  KDB_TRY(validate_eps(eps));
  if (M < 1 || M > g->k_max) return set_err(KDB_EINVAL, "M must be in [1, k_max]");
  if (!core_bits && g->n_total > 0) return set_err(KDB_EINVAL, "core_bits is NULL");
  if (comm && comm->kind == 2 && (g->row_begin != 0 || g->n_rows != g->n_total))
    return set_err(KDB_EINVAL, "sim communicator needs the full graph");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nwords = (g->n_total + 31) / 32;
  if (nwords == 0) return KDB_OK;
  KDB_CUDA(cudaMemsetAsync(core_bits, 0, nwords * sizeof(uint32_t), st));
  std::vector<int64_t> rb, rn;
  rank_ranges(g, comm, rb, rn);
  for (size_t r = 0; r < rb.size(); ++r) {
    if (rn[r] == 0) continue;
    const int64_t off = (rb[r] - g->row_begin) * g->k_max;
    LAUNCH(k_core_mark, grid_for(rn[r] / 32 + 2), kThreads, st, g->dist + off, rn[r], g->k_max, M, eps, rb[r], core_bits);
    KDB_CUDA(cudaGetLastError());
  }
  // ranks own disjoint bits: SUM == OR
  if (multi_rank(comm))
    KDB_TRY(nccl_check(g_nccl.AllReduce(core_bits, core_bits, (size_t)nwords, ncclUint32, ncclSum,
                                        comm->nccl, st), "ncclAllReduce(core bits)"));
  if (g_prof.on) {  // profiling mode only: resolve timings now (synchronises)
    KDB_CUDA(cudaStreamSynchronize(st));
    g_prof.drain();
  }
  return KDB_OK;
}

int32_t edge_cols_of(const kdb_graph* g) {
  return (g->edge_cols > 0 && g->edge_cols < g->k_max) ? g->edge_cols : g->k_max;
}

size_t kdb_mst_workspace_bytes(const kdb_graph* g, kdb_comm* comm) {
  if (validate_graph(g) != KDB_OK) return 0;
  std::vector<int64_t> rb, rn;
  rank_ranges(g, comm, rb, rn);
  Layout L;
  return carve(L, nullptr, true, g->n_total, (int)rb.size(), rb.data(), rn.data(), !(g->flags & KDB_GRAPH_EXACT),
               edge_cols_of(g));
}

}  // extern "C"
namespace {
// bytes of the inexact mode's local view (nbr + dist copies of the rows)
size_t local_view_bytes(const kdb_graph* g) {
  return 2 * (((size_t)g->n_rows * g->k_max * 4 + 255) & ~size_t(255));
}
// kdb_mst (nparts = 0) and kdb_mst_inexact (nparts >= 1 contiguous groups)
kdb_status mst_impl(const kdb_graph* g, float eps, const uint32_t* core_bits, int32_t* comp, uint32_t* mst_a,
                    uint32_t* mst_b, float* mst_w, int64_t mst_cap, int64_t* mst_count, double* mst_weight,
                    void* workspace, size_t ws_bytes, kdb_comm* comm, kdb_stream_t stream, int32_t nparts) {
  KDB_TRY(validate_graph(g));
  KDB_TRY(validate_eps(eps));
  const int64_t N = g->n_total;
  if (!mst_count || !mst_weight) return set_err(KDB_EINVAL, "mst_count/mst_weight is NULL");
  if (N > 0 && (!core_bits || !comp || !workspace)) return set_err(KDB_EINVAL, "NULL device pointer");
  if (mst_cap < 0 || (mst_cap > 0 && (!mst_a || !mst_b || !mst_w)))
    return set_err(KDB_EINVAL, "bad MSF output arrays");
  if (comm && comm->kind == 2 && (g->row_begin != 0 || g->n_rows != g->n_total))
    return set_err(KDB_EINVAL, "sim communicator needs the full graph");
  if ((uintptr_t)workspace & 255u) return set_err(KDB_EINVAL, "workspace must be 256-byte aligned");
  const bool inexact = nparts > 0;
  if (inexact && (comm || g->row_begin != 0 || g->n_rows != g->n_total))
    return set_err(KDB_EINVAL, "kdb_mst_inexact: single process, full graph");
  int32_t* lnbr = nullptr;
  float* ldist = nullptr;
  if (inexact) {  // the local view leads the workspace
    const size_t lv = local_view_bytes(g);
    if (ws_bytes < lv) return set_err(KDB_ENOMEM, "workspace %zu < required %zu bytes", ws_bytes, lv);
    lnbr = reinterpret_cast<int32_t*>(workspace);
    ldist = reinterpret_cast<float*>((char*)workspace + lv / 2);
    workspace = (char*)workspace + lv;
    ws_bytes -= lv;
  }
  Mst m;
  m.g = g;
  m.comm = comm;
  m.st = (cudaStream_t)stream;
  m.N = N;
  m.k = edge_cols_of(g);  // kernels stride rows by ld and take candidates from columns < k
  m.ld = g->k_max;
  m.bits = core_bits;
  m.comp = comp;
  // the local view is no kNN graph (no certificate): in-edge lists
  m.general = inexact || !(g->flags & KDB_GRAPH_EXACT);
  Layout& L = m.L;
  std::vector<int64_t> rb, rn;
  rank_ranges(g, comm, rb, rn);
  const size_t need = carve(L, (char*)workspace, false, N, (int)rb.size(), rb.data(), rn.data(), m.general, m.k,
                            inexact ? g->n_rows * (int64_t)m.k : -1);
  if (ws_bytes < need) return set_err(KDB_ENOMEM, "workspace %zu < required %zu bytes", ws_bytes, need);
  *mst_count = 0;
  *mst_weight = 0.0;
  for (auto& s : g_stats) s = 0;
  if (N == 0) return KDB_OK;
  cudaStream_t st = m.st;
  for (auto& R : L.ranks) {
    R.nbr = g->nbr + (R.row_begin - g->row_begin) * m.ld;
    R.dist = g->dist + (R.row_begin - g->row_begin) * m.ld;
  }
  for (auto& e : m.ev) KDB_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() { for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]); }
  } guard{m.ev};

  // Filter-Boruvka when a light threshold below eps exists;
  // plain rows-Boruvka over the whole candidate graph otherwise.
  const int light_m = env_int("KDB_LIGHT", 10);
  bool filtered = false;
  if (inexact) {
    // U_i MST_i,local: the rows phase on the local view; then MST_cut: the cut
    // entries of the real rows as survivors between local components
    RankState& R = L.ranks[0];
    LAUNCH(k_local_view, grid_for(N), kThreads, st, g->nbr, g->dist, N, m.ld, m.k, (int)nparts, lnbr, ldist);
    R.nbr = lnbr;
    R.dist = ldist;
    KDB_TRY(rows_phase(m, eps));
    KDB_CUDA(cudaEventRecord(m.ev[0], st));
    KDB_CUDA(cudaMemsetAsync(R.n_hs_dev, 0, 2 * sizeof(uint32_t), st));
    LAUNCH(k_cut_edges, grid_for(N), kThreads, st, g->nbr, g->dist, N, m.ld, m.k, eps, (int)nparts, core_bits,
           comp, R.hs[0], R.hs_cap, R.n_hs_dev);
    KDB_CUDA(cudaGetLastError());
    uint32_t ncut = 0;
    KDB_CUDA(cudaMemcpyAsync(&ncut, R.n_hs_dev, 4, cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    if (ncut > R.hs_cap) return set_err(KDB_EINTERNAL, "cut entries exceed their buffer");
    R.n_hs = ncut;
    m.survivors = ncut;
    KDB_CUDA(cudaEventRecord(m.ev[1], st));
    m.t_filter += elapsed(m.ev[0], m.ev[1]);
    KDB_TRY(heavy_phase(m));
  } else if (env_int("KDB_FILTER", 1) && light_m >= 1 && light_m < m.k) {
    KDB_TRY(pick_tau(m, light_m, &m.tau));
    filtered = m.tau < eps;
  }
  if (inexact) {
    // done above
  } else if (filtered) {
    KDB_TRY(rows_phase(m, m.tau));
    bool overflow = false;
    KDB_TRY(filter_phase(m, eps, &overflow));
    if (overflow) {  // too many crossing heavy entries for the survivor buffers
      m.fallback = 1;
      m.C_heavy = -1;
      KDB_TRY(rows_phase(m, eps));
    } else {
      KDB_TRY(heavy_phase(m));
    }
  } else {
    KDB_TRY(rows_phase(m, eps));
  }

  // ---- finalize ---------------------------------------------------------------------
  KDB_CUDA(cudaEventRecord(m.ev[0], st));
  RoundCounters hc;
  KDB_CUDA(cudaMemcpyAsync(&hc, L.ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
  KDB_CUDA(cudaStreamSynchronize(st));
  const int64_t ne = (int64_t)hc.msf_count;
  if (ne > N) return set_err(KDB_EINTERNAL, "MSF larger than N-1");
  if (ne > mst_cap) return set_err(KDB_EINVAL, "mst_cap %lld < MSF size %lld", (long long)mst_cap, (long long)ne);
  // canonical labels: comp[v] = cmin[comp[v]] (through hcomp after a heavy phase)
  if (m.C_heavy >= 0)
    LAUNCH(k_relabel, grid_for(N / 8 + 1), kThreads, st, N, comp, L.hcomp, L.cmin);
  else
    LAUNCH(k_relabel, grid_for(N / 8 + 1), kThreads, st, N, comp, L.cmin, (const int32_t*)nullptr);
  KDB_CUDA(cudaGetLastError());
  unsigned long long bk[256];
  if (ne > 0) {
    size_t cb = L.cub_bytes;
    unsigned long long* vb2 = reinterpret_cast<unsigned long long*>(L.Kc);  // N + 1, free now
    int abits = 1;
    while (abits < 32 && ((int64_t)1 << abits) < N) ++abits;
    {
      // the emitted (a, (b, w)) pairs sort straight into the caller's mst_a
      LaunchScope ls_("cub::DeviceRadixSort", st, false);
      KDB_CUDA(cub::DeviceRadixSort::SortPairs(L.cub_tmp, cb, reinterpret_cast<const uint32_t*>(L.e_w), mst_a,
                                               reinterpret_cast<const unsigned long long*>(L.e_key), vb2, (int)ne, 0,
                                               abits, st));
    }
    LAUNCH(k_msf_unpack, grid_for(ne), kThreads, st, ne, mst_a, vb2, mst_b, mst_w);
    KDB_CUDA(cudaMemsetAsync(L.buckets, 0, 256 * sizeof(unsigned long long), st));
    LAUNCH(k_wbuckets, grid_for(ne), kThreads, st, ne, mst_w, L.buckets);
    KDB_CUDA(cudaGetLastError());
    KDB_CUDA(cudaMemcpyAsync(bk, L.buckets, sizeof(bk), cudaMemcpyDeviceToHost, st));
  }
  KDB_CUDA(cudaEventRecord(m.ev[1], st));
  KDB_CUDA(cudaStreamSynchronize(st));
  const double t_fin = elapsed(m.ev[0], m.ev[1]);
  if (g_prof.on) g_prof.drain();
  *mst_count = ne;
  *mst_weight = ne > 0 ? exact_bucket_sum(bk) : 0.0;
  g_stats[0] = m.rounds;
  g_stats[1] = m.t_init;
  g_stats[2] = m.t_min_edges;
  g_stats[3] = m.t_contract;
  g_stats[4] = t_fin;
  g_stats[5] = m.t_inlist;
  g_stats[6] = m.stalls;
  g_stats[7] = (double)m.entries;
  g_stats[8] = m.t_filter;
  g_stats[9] = m.t_heavy;
  g_stats[10] = (double)m.survivors;
  g_stats[11] = m.heavy_rounds;
  g_stats[12] = filtered ? (double)m.tau : -1.0;
  g_stats[13] = (double)m.C;
  g_stats[14] = m.fallback;
  g_stats[15] = (double)m.exceptions;
  g_stats[16] = (double)m.slow_entries;
  g_stats[17] = inexact ? 0.0 : m.payload_rows;  // inexact: the groups' local phases share nothing
  g_stats[18] = m.payload_heavy;
  return KDB_OK;
}

}  // namespace
extern "C" {

kdb_status kdb_mst(const kdb_graph* g, float eps, const uint32_t* core_bits, int32_t* comp,
                   uint32_t* mst_a, uint32_t* mst_b, float* mst_w, int64_t mst_cap, int64_t* mst_count,
                   double* mst_weight, void* workspace, size_t ws_bytes, kdb_comm* comm,
                   kdb_stream_t stream) {
  return mst_impl(g, eps, core_bits, comp, mst_a, mst_b, mst_w, mst_cap, mst_count, mst_weight, workspace, ws_bytes,
                  comm, stream, 0);
}

size_t kdb_mst_inexact_workspace_bytes(const kdb_graph* g, int32_t nparts) {
  if (validate_graph(g) != KDB_OK || nparts < 1) return 0;
  std::vector<int64_t> rb{g->row_begin}, rn{g->n_rows};
  Layout L;
  return local_view_bytes(g) + carve(L, nullptr, true, g->n_total, 1, rb.data(), rn.data(), true, edge_cols_of(g),
                                     g->n_rows * (int64_t)edge_cols_of(g));
}

kdb_status kdb_mst_inexact(const kdb_graph* g, float eps, const uint32_t* core_bits, int32_t nparts, int32_t* comp,
                           uint32_t* mst_a, uint32_t* mst_b, float* mst_w, int64_t mst_cap, int64_t* mst_count,
                           double* mst_weight, void* workspace, size_t ws_bytes, kdb_stream_t stream) {
  if (nparts < 1) return set_err(KDB_EINVAL, "nparts must be >= 1");
  return mst_impl(g, eps, core_bits, comp, mst_a, mst_b, mst_w, mst_cap, mst_count, mst_weight, workspace, ws_bytes,
                  nullptr, stream, nparts);
}

kdb_status kdb_label(const kdb_graph* g, float eps, const uint32_t* core_bits, const int32_t* comp,
                     int32_t* labels, kdb_stream_t stream) {
  KDB_TRY(validate_graph(g));
  KDB_TRY(validate_eps(eps));
  if (g->n_rows > 0 && (!core_bits || !comp || !labels)) return set_err(KDB_EINVAL, "NULL device pointer");
  if (g->n_rows == 0) return KDB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (g->k_max % 4 == 0)
    LAUNCH(k_label<true>, grid_for(g->n_rows), kThreads, st, g->nbr, g->dist, g->n_rows, g->k_max, eps,
           g->row_begin, g->n_total, core_bits, comp, labels);
  else
    LAUNCH(k_label<false>, grid_for(g->n_rows), kThreads, st, g->nbr, g->dist, g->n_rows, g->k_max, eps,
           g->row_begin, g->n_total, core_bits, comp, labels);
  KDB_CUDA(cudaGetLastError());
  if (g_prof.on) {
    KDB_CUDA(cudaStreamSynchronize(st));
    g_prof.drain();
  }
  return KDB_OK;
}


// ============================================================================
// Clustering quality: NMI and cluster counts
// ============================================================================
// NMI = 2 I / (H(A) + H(B)) with NOISE as one pseudo-cluster per labelling
// (the paper reports NMI without a formula).
// With S_x = sum over the cells of a histogram of n ln n:
//   H(A) = ln N - S_a / N,  I = (S_ab + N ln N - S_a - S_b) / N.
// The histograms are run lengths of sorted keys (label + 1: NOISE -> 0).
}  // extern "C"
namespace {
__global__ void k_nmi_keys(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n, int bb,
                           uint64_t* __restrict__ pk, uint32_t* __restrict__ ka, uint32_t* __restrict__ kb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = (uint32_t)(a[i] + 1), y = (uint32_t)(b[i] + 1);
    pk[i] = ((uint64_t)x << bb) | y;
    ka[i] = x;
    kb[i] = y;
  }
}
// f[i] = c ln c for the run lengths c of one histogram
__global__ void k_nlogn(const int32_t* __restrict__ cnt, const int32_t* __restrict__ n_runs, double* __restrict__ out) {
  const int m = *n_runs;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const double c = (double)cnt[i];
    out[i] = c * log(c);
  }
}
struct NmiWs {
  uint64_t *k0, *k1, *uniq;
  int32_t* cnt;
  double* f;
  int32_t* runs;
  double* sum;
  int32_t* mm;  // min a, max a, min b, max b
  void* tmp;
  size_t tmp_bytes;
};
size_t nmi_carve(NmiWs& w, char* base, bool dry, int64_t n) {
  Carver cv{base, 0, 0, dry};
  const int64_t m = std::max<int64_t>(n, 1);
  w.k0 = cv.take<uint64_t>(m);
  w.k1 = cv.take<uint64_t>(m);
  w.uniq = cv.take<uint64_t>(m);
  w.cnt = cv.take<int32_t>(m);
  w.f = cv.take<double>(m);
  w.runs = cv.take<int32_t>(4);
  w.sum = cv.take<double>(4);
  w.mm = cv.take<int32_t>(4);
  size_t t = 0, x = 0;
  const int ni = (int)m;
  cub::DeviceRadixSort::SortKeys(nullptr, x, (const uint64_t*)nullptr, (uint64_t*)nullptr, ni);
  t = std::max(t, x);
  cub::DeviceRadixSort::SortKeys(nullptr, x, (const uint32_t*)nullptr, (uint32_t*)nullptr, ni);
  t = std::max(t, x);
  cub::DeviceRunLengthEncode::Encode(nullptr, x, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int32_t*)nullptr,
                                     (int32_t*)nullptr, ni);
  t = std::max(t, x);
  cub::DeviceRunLengthEncode::Encode(nullptr, x, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int32_t*)nullptr,
                                     (int32_t*)nullptr, ni);
  t = std::max(t, x);
  cub::DeviceReduce::Sum(nullptr, x, (const double*)nullptr, (double*)nullptr, ni);
  t = std::max(t, x);
  cub::DeviceReduce::Min(nullptr, x, (const int32_t*)nullptr, (int32_t*)nullptr, ni);
  t = std::max(t, x);
  cub::DeviceReduce::Max(nullptr, x, (const int32_t*)nullptr, (int32_t*)nullptr, ni);
  t = std::max(t, x);
  w.tmp_bytes = t;
  w.tmp = cv.take<char>(t);
  return cv.off + 256;
}
int bits_for(uint64_t v) {
  int b = 1;
  while (b < 64 && (v >> b)) ++b;
  return b;
}
// run lengths of the sorted keys (T = u32 / u64) -> w.cnt, their count -> w.runs[slot], c ln c -> w.f
template <typename T>
kdb_status nmi_hist(NmiWs& w, const T* sorted, int64_t n, int slot, cudaStream_t st) {
  size_t tb = w.tmp_bytes;
  {
    LaunchScope ls_("cub::DeviceRunLengthEncode", st, false);
    KDB_CUDA(cub::DeviceRunLengthEncode::Encode(w.tmp, tb, sorted, reinterpret_cast<T*>(w.uniq), w.cnt,
                                                w.runs + slot, (int)n, st));
  }
  LAUNCH(k_nlogn, grid_for(n), kThreads, st, w.cnt, w.runs + slot, w.f);
  KDB_CUDA(cudaGetLastError());
  return KDB_OK;
}
}  // namespace
extern "C" {

size_t kdb_nmi_workspace_bytes(int64_t n) {
  if (n < 0 || n >= (int64_t)INT32_MAX) return 0;
  NmiWs w;
  return nmi_carve(w, nullptr, true, n);
}

kdb_status kdb_nmi(const int32_t* a, const int32_t* b, int64_t n, double* nmi, int64_t* clusters_a,
                   int64_t* clusters_b, void* workspace, size_t ws_bytes, kdb_stream_t stream) {
  if (!nmi || !clusters_a || !clusters_b) return set_err(KDB_EINVAL, "NULL host output");
  if (n < 0 || n >= (int64_t)INT32_MAX) return set_err(KDB_EINVAL, "n out of range [0, 2^31-1)");
  if (n > 0 && (!a || !b || !workspace)) return set_err(KDB_EINVAL, "NULL device pointer");
  if ((uintptr_t)workspace & 255u) return set_err(KDB_EINVAL, "workspace must be 256-byte aligned");
  NmiWs w;
  const size_t need = nmi_carve(w, (char*)workspace, false, n);
  if (n > 0 && ws_bytes < need) return set_err(KDB_ENOMEM, "workspace %zu < required %zu bytes", ws_bytes, need);
  *nmi = 1.0;
  *clusters_a = *clusters_b = 0;
  if (n == 0) return KDB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int ni = (int)n;
  size_t tb = w.tmp_bytes;
  {
    LaunchScope ls_("cub::DeviceReduce", st, false);
    KDB_CUDA(cub::DeviceReduce::Min(w.tmp, tb, a, w.mm + 0, ni, st));
    KDB_CUDA(cub::DeviceReduce::Max(w.tmp, tb, a, w.mm + 1, ni, st));
    KDB_CUDA(cub::DeviceReduce::Min(w.tmp, tb, b, w.mm + 2, ni, st));
    KDB_CUDA(cub::DeviceReduce::Max(w.tmp, tb, b, w.mm + 3, ni, st));
  }
  int32_t mm[4];
  KDB_CUDA(cudaMemcpyAsync(mm, w.mm, sizeof(mm), cudaMemcpyDeviceToHost, st));
  KDB_CUDA(cudaStreamSynchronize(st));
  if (mm[0] < -1 || mm[2] < -1) return set_err(KDB_EINVAL, "labels must be >= -1 (NOISE)");
  const int ba = bits_for((uint64_t)mm[1] + 1), bb = bits_for((uint64_t)mm[3] + 1);
  // pair keys -> k0; a + 1 -> f (first n u32); b + 1 -> f (next n u32)
  uint32_t* sa = reinterpret_cast<uint32_t*>(w.f);
  uint32_t* sb = sa + n;
  LAUNCH(k_nmi_keys, grid_for(n), kThreads, st, a, b, n, bb, w.k0, sa, sb);
  KDB_CUDA(cudaGetLastError());
  double S[3];
  int32_t runs[3];
  uint32_t first[3];
  for (int pass = 0; pass < 3; ++pass) {
    tb = w.tmp_bytes;
    if (pass == 0) {
      {
        LaunchScope ls_("cub::DeviceRadixSort", st, false);
        KDB_CUDA(cub::DeviceRadixSort::SortKeys(w.tmp, tb, w.k0, w.k1, ni, 0, std::min(64, ba + bb), st));
      }
      // the single-label keys move to k0 (free now) before f is overwritten
      KDB_CUDA(cudaMemcpyAsync(w.k0, sa, 2 * n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
      KDB_TRY(nmi_hist<uint64_t>(w, w.k1, n, 0, st));
    } else {
      uint32_t* src = reinterpret_cast<uint32_t*>(w.k0) + (pass == 1 ? 0 : n);
      uint32_t* dst = reinterpret_cast<uint32_t*>(w.k1);
      {
        LaunchScope ls_("cub::DeviceRadixSort", st, false);
        KDB_CUDA(cub::DeviceRadixSort::SortKeys(w.tmp, tb, src, dst, ni, 0, pass == 1 ? ba : bb, st));
      }
      KDB_TRY(nmi_hist<uint32_t>(w, dst, n, pass, st));
    }
    KDB_CUDA(cudaMemcpyAsync(&runs[pass], w.runs + pass, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaMemcpyAsync(&first[pass], w.uniq, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    tb = w.tmp_bytes;
    {
      LaunchScope ls_("cub::DeviceReduce", st, false);
      KDB_CUDA(cub::DeviceReduce::Sum(w.tmp, tb, w.f, w.sum + pass, runs[pass], st));
    }
    KDB_CUDA(cudaMemcpyAsync(&S[pass], w.sum + pass, sizeof(double), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
  }
  const double N = (double)n, lnN = log(N);
  const double Ha = lnN - S[1] / N, Hb = lnN - S[2] / N;
  const double I = (S[0] + N * lnN - S[1] - S[2]) / N;
  const bool za = runs[1] == 1, zb = runs[2] == 1;  // a single cell: zero entropy (exactly)
  if (za && zb) *nmi = 1.0;
  else if (za || zb) *nmi = 0.0;
  else *nmi = std::min(1.0, std::max(0.0, 2.0 * I / (Ha + Hb)));
  // the smallest key is NOISE + 1 = 0 iff the labelling has noise
  *clusters_a = runs[1] - (first[1] == 0u ? 1 : 0);
  *clusters_b = runs[2] - (first[2] == 0u ? 1 : 0);
  return KDB_OK;
}

}  // extern "C"
