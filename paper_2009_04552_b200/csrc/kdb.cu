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
thread_local double g_stats[8];

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
  (void)0;
  int64_t g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  // grid-stride kernels: at most one resident wave (8 x 256-thread CTAs per SM);
  // a second wave would only start after the first finished ALL its strides
  const int cap = getenv("KDB_GRIDCAP") ? atoi(getenv("KDB_GRIDCAP")) : 148 * 8;
  if (g > cap) g = cap;
  return (int)g;
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
const int g_sortcont = getenv("KDB_SORTCONT") ? atoi(getenv("KDB_SORTCONT")) : 0;
const int g_lines = getenv("KDB_LINES") ? atoi(getenv("KDB_LINES")) : 4;
const int g_fa = getenv("KDB_FA") ? atoi(getenv("KDB_FA")) : 1;  // first block lines, awake rows
const int g_fs = getenv("KDB_FS") ? atoi(getenv("KDB_FS")) : 4;  // first block lines, woken rows
const int g_lazy = getenv("KDB_LAZY") ? atoi(getenv("KDB_LAZY")) : 1;
const int g_qmax = getenv("KDB_QMAX") ? atoi(getenv("KDB_QMAX")) : 1;
const uint32_t g_chunk = getenv("KDB_CHUNK") ? (uint32_t)atoi(getenv("KDB_CHUNK")) : (1u << 30);
const uint32_t g_chunk_w = getenv("KDB_CHUNKW") ? (uint32_t)atoi(getenv("KDB_CHUNKW")) : (1u << 30);

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
#define LAUNCH(kern, grid, block, st, ...)             \
  do {                                                 \
    LaunchScope ls_(#kern, st);                        \
    kern<<<(grid), (block), 0, (st)>>>(__VA_ARGS__);   \
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
  uint32_t part[2];              // next round: awake rows, asleep rows
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
__global__ void k_core_mark(const float* __restrict__ dist, int64_t n_rows, int32_t k, int32_t M,
                            float eps, int64_t row_begin, uint32_t* __restrict__ bits) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_rows;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool in = i < n_rows;
    bool core = false;
    if (in) core = __ldcs(dist + i * k + (M - 1)) <= eps;
    const int64_t v = row_begin + i;
    const unsigned inmask = __ballot_sync(0xffffffffu, in);
    if (in) {
      const unsigned grp = __match_any_sync(inmask, (unsigned long long)(v >> 5));
      const unsigned word = __reduce_or_sync(grp, core ? (1u << (v & 31)) : 0u);
      if ((threadIdx.x & 31) == __ffs(grp) - 1 && word) atomicOr(bits + (v >> 5), word);
    }
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
                                   uint32_t* __restrict__ kmin) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    Kc[c] = kSent;
    Bc[c] = kSentB;
    if (kmin) kmin[c] = kInfBits;
  }
}

// ---------------------------------------------------------------------------
// Active-row records.  The scan position L[i] travels with the
// row id through the active lists, so a row's state arrives in one coalesced
// 8-byte load instead of a chain of dependent gathers.
struct Act {
  int32_t v;   // global row id
  int32_t h;   // head: every entry before it is dead for good
  float lb;    // asleep rows: every live entry at/after h weighs >= lb
  int32_t asleep;  // 1: deferred -- skipped by pass A, only wake-checked
};
// continuation record: everything k_offer_warp needs, written by k_offer_rows_t
struct Cont {
  int32_t v, h, cv, s;  // row, head, its component, slot in the active list
};

// local rows: certificate bound kth'(v) into kmin[comp v], active list (v, head 0)
__global__ void k_init_rows(const float* __restrict__ dist, int64_t n_rows, int32_t k, float eps,
                            int64_t row_begin, const uint32_t* __restrict__ bits,
                            const int32_t* __restrict__ comp, uint32_t* __restrict__ kmin,
                            Act* __restrict__ active, uint8_t* __restrict__ flag) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_rows;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool want = false;
    int64_t v = row_begin + i;
    if (i < n_rows) {
      if (is_core(bits, v)) {
        // a row whose first entry is already beyond eps offers nothing, ever
        want = __ldcs(dist + i * k) <= eps;
        if (kmin) {
          const float kth = __ldcs(dist + i * k + (k - 1));
          kmin[comp[v]] = (kth <= eps) ? mono_bits(kth) : kInfBits;
        }
      }
    }
    if (i < n_rows) {
      active[i] = Act{(int32_t)v, 0, 0.f, 0};  // awake
      flag[i] = want ? 1 : 0;
    }
  }
}

// ============================================================================
// general mode: in-edge lists (transpose of local candidate entries)
// ============================================================================
__global__ void k_in_count(const int32_t* __restrict__ nbr, const float* __restrict__ dist,
                           int64_t n_rows, int32_t k, float eps, int64_t row_begin, int64_t N,
                           const uint32_t* __restrict__ bits, unsigned long long* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = row_begin + i;
    if (!is_core(bits, v)) continue;
    for (int32_t c = 0; c < k; ++c) {
      const float w = __ldg(dist + i * k + c);
      if (!(w <= eps)) break;
      const int64_t J = __ldg(nbr + i * k + c);
      if (J < 0 || J >= N || J == v || !is_core(bits, J)) continue;
      atomicAdd(cnt + J, 1ull);
    }
  }
}

__global__ void k_in_fill(const int32_t* __restrict__ nbr, const float* __restrict__ dist,
                          int64_t n_rows, int32_t k, float eps, int64_t row_begin, int64_t N,
                          const uint32_t* __restrict__ bits, unsigned long long* __restrict__ cursor,
                          int32_t* __restrict__ in_src, float* __restrict__ in_w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = row_begin + i;
    if (!is_core(bits, v)) continue;
    for (int32_t c = 0; c < k; ++c) {
      const float w = __ldg(dist + i * k + c);
      if (!(w <= eps)) break;
      const int64_t J = __ldg(nbr + i * k + c);
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
// (after skipping permanently dead entries) whose far endpoint lies in another
// component opens the minimum group; equal-weight entries after it may carry a
// smaller far id and are scanned too.  The head pointer only passes entries
// that can never become leaving again (non-candidates, intra-component).
//
__device__ __forceinline__ bool cand_entry(int64_t J, int64_t v, int64_t N, const uint32_t* bits, bool all_core) {
  return J >= 0 && J < N && J != v && (all_core || is_core(bits, J));
}

// One thread per active row; each step takes an aligned 4-entry chunk (int4
// ids + float4 weights when k % 4 == 0, loaded evict-first so the streamed
// graph does not push comp[] out of L2) and issues its 4 component gathers
// together.  A thread gives up after qmax chunks of dead entries (the chunk
// count per row varies 1..k/4 inside a warp); the row then continues in
// k_offer_warp, 32 entries per step.

template <bool VEC>
__device__ __forceinline__ void load_chunk(const int32_t* nr, const float* dr, int c0, int k, int32_t (&J)[4],
                                           float (&w)[4]) {
  if (VEC && c0 + 3 < k) {
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

template <bool VEC>
__global__ void __launch_bounds__(256) k_offer_rows_t(
    const int32_t* __restrict__ nbr, const float* __restrict__ dist, int32_t k, float eps, int64_t row_begin,
    int64_t N, const uint32_t* __restrict__ bits, int all_core, const int32_t* __restrict__ comp,
    Act* __restrict__ act, uint32_t s_begin, uint32_t s_end, uint8_t* __restrict__ status,
    uint64_t* __restrict__ off_key, uint32_t* __restrict__ off_b, Cont* __restrict__ cand,
    unsigned long long* __restrict__ Kc, unsigned long long* __restrict__ n_entries, int qmax) {
  unsigned long long reads = 0;
  for (uint32_t s = s_begin + blockIdx.x * blockDim.x + threadIdx.x; s < s_end; s += gridDim.x * blockDim.x) {
    bool found = false, more = false;
    uint64_t best = kSent;
    uint32_t bestb = kSentB;
    const int4 a = __ldcs(reinterpret_cast<const int4*>(act + s));
    if (a.w) continue;  // asleep: k_wake decides
    const int32_t v = a.x;
    int h = a.y;
    const int64_t i = (int64_t)v - row_begin;
    const int32_t* nr = nbr + i * k;
    const float* dr = dist + i * k;
    const int32_t cv = gat(comp + v);
    int c0 = h & ~3;
    float wstar = 0.f, wlast = 0.f;  // wlast: weight of the last dead entry passed
    bool done = false;
    int steps = 0;
    while (!done && c0 < k) {
      if (!found && steps == qmax) {  // hand the rest of the dead run to a warp
        more = true;
        break;
      }
      ++steps;
      int32_t J[4];
      float w[4];
      load_chunk<VEC>(nr, dr, c0, k, J, w);
      int32_t cj[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool ok = c0 + j >= h && w[j] <= eps && cand_entry(J[j], v, N, bits, all_core);
        cj[j] = ok ? gat(comp + J[j]) : -2;  // -2: not a candidate (dead for good)
      }
      reads += (unsigned long long)(min(c0 + 4, k) - max(c0, h));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int idx = c0 + j;
        if (done || idx < h || idx >= k) continue;
        if (!found) {
          if (!(w[j] <= eps)) { h = k; done = true; continue; }  // sorted: nothing left
          if (cj[j] == -2 || cj[j] == cv) { h = idx + 1; wlast = w[j]; continue; }  // dead entry
          found = true;  // first leaving entry opens the minimum group
          h = idx;
          wstar = w[j];
          best = pack_key(mono_bits(w[j]), (uint32_t)min((int64_t)v, (int64_t)J[j]));
          bestb = (uint32_t)max((int64_t)v, (int64_t)J[j]);
        } else {
          if (w[j] != wstar) { done = true; continue; }
          if (cj[j] == -2 || cj[j] == cv) continue;
          const uint64_t kk = pack_key(mono_bits(w[j]), (uint32_t)min((int64_t)v, (int64_t)J[j]));
          const uint32_t bb = (uint32_t)max((int64_t)v, (int64_t)J[j]);
          if (kk < best || (kk == best && bb < bestb)) { best = kk; bestb = bb; }
        }
      }
      c0 += 4;
    }
    h = min(h, k);
    act[s].h = h;
    __stcs(status + s, (uint8_t)(found ? 1 : (more ? 2 : 0)));  // 1 offer, 2 continue, 0 exhausted
    if (found) {
      __stcs(reinterpret_cast<unsigned long long*>(off_key) + s, (unsigned long long)best);
      __stcs(off_b + s, bestb);
      atomicMin(Kc + cv, (unsigned long long)best);
    } else if (more) {
      if (cand) __stcs(reinterpret_cast<int4*>(cand + s), make_int4(v, h, cv, (int)s));
      act[s].lb = wlast;  // every leaving entry still ahead weighs >= wlast (rows are sorted)
    }
  }
  for (int o = 16; o > 0; o >>= 1) reads += __shfl_xor_sync(0xffffffffu, reads, o);
  if ((threadIdx.x & 31) == 0 && reads) atomicAdd(n_entries, reads);
}

// Continuation: one warp per row.  Lane l takes entries h+l, h+l+32, h+l+64,
// h+l+96 of a 128-entry block: all id/weight loads and all component gathers
// of the block are in flight together (no dependency between lines), then the
// warp reduces (first leaving position, minimum key of the equal-weight group
// that starts there).  Rows are sorted, so the minimum over the block's
// leaving entries with the smallest weight IS that group's minimum; only when a
// group reaches the end of the block does the next block have to be looked at.
template <int kLines>
__global__ void __launch_bounds__(256) k_offer_warp(
    const int32_t* __restrict__ nbr, const float* __restrict__ dist, int32_t k, float eps, int64_t row_begin,
    int64_t N, const uint32_t* __restrict__ bits, int all_core, const int32_t* __restrict__ comp,
    const Cont* __restrict__ cont, const uint32_t* __restrict__ n_cont_p, uint32_t q_begin, uint32_t q_end,
    Act* __restrict__ act, uint8_t* __restrict__ status, uint64_t* __restrict__ off_key,
    uint32_t* __restrict__ off_b, unsigned long long* __restrict__ Kc, unsigned long long* __restrict__ n_entries) {
  const int lane = threadIdx.x & 31;
  const uint32_t n_cont = min(*n_cont_p, q_end);
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  unsigned long long reads = 0;
  uint32_t q = q_begin + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int4 rec = make_int4(0, 0, 0, 0);
  if (q < n_cont) rec = __ldcs(reinterpret_cast<const int4*>(cont + q));
  for (; q < n_cont; q += nwarps) {
    const int32_t v = rec.x, cv = rec.z, s = rec.w;
    const int h0 = rec.y;
    if (q + nwarps < n_cont) rec = __ldcs(reinterpret_cast<const int4*>(cont + q + nwarps));
    const int64_t i = (int64_t)v - row_begin;
    const int32_t* nr = nbr + i * k;
    const float* dr = dist + i * k;
    int pos = k;              // first leaving position found so far
    uint32_t wbest = 0xffffffffu;  // its weight bits
    uint64_t best = kSent;
    uint32_t bestb = kSentB;
    int base = h0;
    bool stop = false;
    while (!stop && base < k) {
      float w[kLines];
      int32_t J[kLines];
#pragma unroll
      for (int t = 0; t < kLines; ++t) {
        const int c = base + lane + 32 * t;
        w[t] = c < k ? __ldcs(dr + c) : __int_as_float(0x7f800000);
        J[t] = c < k ? __ldcs(nr + c) : -1;
      }
      int32_t cj[kLines];
#pragma unroll
      for (int t = 0; t < kLines; ++t)
        cj[t] = (w[t] <= eps && cand_entry(J[t], v, N, bits, all_core)) ? gat(comp + J[t]) : cv;
      bool beyond = false;
      unsigned lp = (unsigned)k;  // this lane's first leaving position in the block
#pragma unroll
      for (int t = kLines - 1; t >= 0; --t) {
        const int c = base + lane + 32 * t;
        if (c < k && !(w[t] <= eps)) beyond = true;
        if (cj[t] != cv) lp = (unsigned)c;
      }
      lp = __reduce_min_sync(0xffffffffu, lp);  // the block's first leaving position
      if ((int)lp < k) {
        if (pos == k) {  // first leaving entry of the row: its weight opens the group
          const int rel = (int)lp - base;
          float wl = 0.f;
#pragma unroll
          for (int t = 0; t < kLines; ++t) {
            const float x = __shfl_sync(0xffffffffu, w[t], rel & 31);
            if ((rel >> 5) == t) wl = x;
          }
          pos = (int)lp;
          wbest = mono_bits(wl);
        }
        // group members in this block: leaving entries of weight wbest; their key's
        // weight part is equal, so the minimum is over (a, b) as two 32-bit mins
        uint32_t am = 0xffffffffu, bm = 0xffffffffu;
#pragma unroll
        for (int t = 0; t < kLines; ++t) {
          const int c = base + lane + 32 * t;
          if (c < k && cj[t] != cv && mono_bits(w[t]) == wbest) {
            const uint32_t a2 = (uint32_t)min((int64_t)v, (int64_t)J[t]);
            const uint32_t b2 = (uint32_t)max((int64_t)v, (int64_t)J[t]);
            if (a2 < am || (a2 == am && b2 < bm)) { am = a2; bm = b2; }
          }
        }
        const uint32_t amin = __reduce_min_sync(0xffffffffu, am);
        const uint32_t bmin = __reduce_min_sync(0xffffffffu, am == amin ? bm : 0xffffffffu);
        const uint64_t kk = pack_key(wbest, amin);
        if (amin != 0xffffffffu && (kk < best || (kk == best && bmin < bestb))) { best = kk; bestb = bmin; }
      }
      bool tail_eq = false;  // an entry of weight wbest sits at the block end
      if (pos < k) {
        const int c = base + lane + 32 * (kLines - 1);
        tail_eq = lane == 31 && c < k && w[kLines - 1] <= eps && mono_bits(w[kLines - 1]) == wbest;
      }
      if (lane == 0) reads += (unsigned long long)(min(base + 32 * kLines, k) - base);
      const bool any_beyond = __any_sync(0xffffffffu, beyond);
      const bool tail = __any_sync(0xffffffffu, tail_eq);
      // stop once a leaving entry was found (unless its group reaches the block
      // end) or the weights passed eps (sorted rows: nothing after)
      stop = any_beyond || (pos < k && !tail);
      base += 32 * kLines;
    }
    if (lane == 0) {
      const bool found = best != kSent;
      act[s].h = found ? pos : k;
      status[s] = found ? 1 : 0;
      if (found) {
        off_key[s] = best;
        off_b[s] = bestb;
        atomicMin(Kc + cv, (unsigned long long)best);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) reads += __shfl_xor_sync(0xffffffffu, reads, o);
  if (lane == 0 && reads) atomicAdd(n_entries, reads);
}

// One warp scans the remaining entries of row v from head h0 (all 32 lanes,
// the whole warp must call it).  Lane l takes entries base+l, base+l+32, ...:
// the first block is one 32-entry line (most rows leave early), later blocks
// are 128 entries with all id/weight loads and component gathers in flight
// together.  Returns (found, first leaving position, minimum key and b of the
// equal-weight group that starts there); rows are sorted, so that group's
// minimum is the row's minimum leaving edge under O1.
struct RowMin {
  bool found;
  int pos;
  uint64_t key;
  uint32_t b;
};

__device__ __forceinline__ RowMin warp_scan_row(const int32_t* __restrict__ nr, const float* __restrict__ dr, int k,
                                                float eps, int32_t v, int32_t cv, int h0, int64_t N,
                                                const uint32_t* __restrict__ bits, int all_core,
                                                const int32_t* __restrict__ comp, unsigned long long& reads,
                                                int first_lines) {
  constexpr int kL = 4;
  const int lane = threadIdx.x & 31;
  int pos = k;
  uint32_t wbest = 0xffffffffu;
  uint64_t best = kSent;
  uint32_t bestb = kSentB;
  int base = h0;
  int lines = first_lines;
  bool stop = false;
  while (!stop && base < k) {
    const int bend = min(base + 32 * lines, k);  // block = [base, bend)
    float w[kL];
    int32_t J[kL];
#pragma unroll
    for (int t = 0; t < kL; ++t) {
      const int c = base + lane + 32 * t;
      const bool in = t < lines && c < bend;
      w[t] = in ? __ldcs(dr + c) : __int_as_float(0x7f800000);
      J[t] = in ? __ldcs(nr + c) : -1;
    }
    int32_t cj[kL];
#pragma unroll
    for (int t = 0; t < kL; ++t)
      cj[t] = (w[t] <= eps && cand_entry(J[t], v, N, bits, all_core)) ? gat(comp + J[t]) : cv;
    bool beyond = false;
    unsigned lp = (unsigned)k;
#pragma unroll
    for (int t = kL - 1; t >= 0; --t) {
      const int c = base + lane + 32 * t;
      if (t < lines && c < bend && !(w[t] <= eps)) beyond = true;
      if (cj[t] != cv) lp = (unsigned)c;
    }
    lp = __reduce_min_sync(0xffffffffu, lp);
    if ((int)lp < k) {
      if (pos == k) {
        const int rel = (int)lp - base;
        float wl = 0.f;
#pragma unroll
        for (int t = 0; t < kL; ++t) {
          const float x = __shfl_sync(0xffffffffu, w[t], rel & 31);
          if ((rel >> 5) == t) wl = x;
        }
        pos = (int)lp;
        wbest = mono_bits(wl);
      }
      uint32_t am = 0xffffffffu, bm = 0xffffffffu;
#pragma unroll
      for (int t = 0; t < kL; ++t) {
        if (cj[t] != cv && mono_bits(w[t]) == wbest) {
          const uint32_t a2 = (uint32_t)min((int64_t)v, (int64_t)J[t]);
          const uint32_t b2 = (uint32_t)max((int64_t)v, (int64_t)J[t]);
          if (a2 < am || (a2 == am && b2 < bm)) { am = a2; bm = b2; }
        }
      }
      const uint32_t amin = __reduce_min_sync(0xffffffffu, am);
      const uint32_t bmin = __reduce_min_sync(0xffffffffu, am == amin ? bm : 0xffffffffu);
      const uint64_t kk = pack_key(wbest, amin);
      if (amin != 0xffffffffu && (kk < best || (kk == best && bmin < bestb))) { best = kk; bestb = bmin; }
    }
    bool tail_eq = false;  // the block's last entry still has the group's weight
    if (pos < k) {
      const int last = bend - 1;
      const int t = (last - base) >> 5;
      if (lane == ((last - base) & 31)) {
#pragma unroll
        for (int u = 0; u < kL; ++u)
          if (u == t) tail_eq = w[u] <= eps && mono_bits(w[u]) == wbest;
      }
    }
    if (lane == 0) reads += (unsigned long long)(bend - base);
    const bool any_beyond = __any_sync(0xffffffffu, beyond);
    const bool tail = __any_sync(0xffffffffu, tail_eq);
    stop = any_beyond || (pos < k && !tail);
    base = bend;
    lines = kL;
  }
  RowMin r;
  r.found = best != kSent;
  r.pos = pos;
  r.key = best;
  r.b = bestb;
  return r;
}

// After pass A: one lane per slot of a 32-slot tile decides whether its row
// must be scanned this round (lazy Boruvka):
//   awake row with a dead first chunk (status 2): scan unless lb > w(Kc[comp])
//     -- then it is deferred (asleep) instead;
//   asleep row: scan (wake) iff lb <= w(Kc[comp]) -- Kc holds an actual
//     leaving edge of the component, so a row whose live entries all weigh
//     more cannot supply the minimum.
// The warp then scans the flagged rows one after another.
__global__ void __launch_bounds__(256) k_scan_tiles(
    const int32_t* __restrict__ nbr, const float* __restrict__ dist, int32_t k, float eps, int64_t row_begin,
    int64_t N, const uint32_t* __restrict__ bits, int all_core, const int32_t* __restrict__ comp,
    Act* __restrict__ act, uint32_t n, uint8_t* __restrict__ status, uint64_t* __restrict__ off_key,
    uint32_t* __restrict__ off_b, unsigned long long* __restrict__ Kc, int lazy,
    unsigned long long* __restrict__ n_entries, uint32_t* __restrict__ n_scanned, int g_first_awake,
    int g_first_asleep) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  unsigned long long reads = 0;
  uint32_t scanned = 0;
  for (uint32_t tile = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; tile * 32 < n; tile += nwarps) {
    const uint32_t s = tile * 32 + lane;
    bool need = false;
    int4 r = make_int4(-1, 0, 0, 0);
    int32_t cv = -1;
    if (s < n) {
      r = __ldcs(reinterpret_cast<const int4*>(act + s));
      const uint8_t st = r.w ? 0xff : status[s];  // 0xff: asleep (pass A skipped it)
      if (st == 2 || st == 0xff) {
        cv = gat(comp + r.x);
        const uint32_t kw = (uint32_t)(gat(Kc + cv) >> 32);  // sentinel -> never deferred
        const bool over = lazy && mono_bits(__int_as_float(r.z)) > kw;
        if (over) {  // cannot supply the minimum this round: (stay) asleep
          status[s] = 4;
          if (!r.w) act[s].asleep = 1;
        } else {
          need = true;
          if (r.w) act[s].asleep = 0;
        }
      }
    }
    unsigned m = __ballot_sync(0xffffffffu, need);
    if (lane == 0) scanned += __popc(m);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const int32_t v = __shfl_sync(0xffffffffu, r.x, src);
      const int32_t h0 = __shfl_sync(0xffffffffu, r.y, src);
      const int32_t c = __shfl_sync(0xffffffffu, cv, src);
      const int32_t was_asleep = __shfl_sync(0xffffffffu, r.w, src);
      const uint32_t ss = tile * 32 + src;
      const int64_t i = (int64_t)v - row_begin;
      // a woken row's first live entry is usually far away; an awake row's is near
      const RowMin rm = warp_scan_row(nbr + i * k, dist + i * k, k, eps, v, c, h0, N, bits, all_core, comp, reads,
                                      was_asleep ? g_first_asleep : g_first_awake);
      if (lane == 0) {
        act[ss].h = rm.found ? rm.pos : k;
        status[ss] = rm.found ? 1 : 0;
        if (rm.found) {
          off_key[ss] = rm.key;
          off_b[ss] = rm.b;
          atomicMin(Kc + c, (unsigned long long)rm.key);
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    reads += __shfl_xor_sync(0xffffffffu, reads, o);
    scanned += __shfl_xor_sync(0xffffffffu, scanned, o);
  }
  if (lane == 0) {
    if (reads) atomicAdd(n_entries, reads);
    if (scanned) atomicAdd(n_scanned, scanned);
  }
}

struct IsTwo {
  __host__ __device__ bool operator()(const uint8_t& x) const { return x == 2; }
};
struct IsOne {
  __host__ __device__ bool operator()(const uint8_t& x) const { return x == 1; }
};
struct IsFour {
  __host__ __device__ bool operator()(const uint8_t& x) const { return x == 4; }
};
struct Survives {  // stays active next round: offered (1) or deferred (4)
  __host__ __device__ bool operator()(const uint8_t& x) const { return x == 1 || x == 4; }
};
struct StatusOf {  // partition predicate over slot indices
  const uint8_t* st;
  uint8_t val;
  __host__ __device__ bool operator()(const int32_t& s) const { return st[s] == val; }
};

// Lazy Boruvka.  A continuing row (status 2) has only dead entries before its
// head and every live entry after it weighs >= lb.  Its component already holds
// an offer Kc (an actual leaving edge, so >= the component's true minimum).  If
// lb > w(Kc) the row cannot supply the minimum this round: defer it (status 4,
// it stays active with its head) instead of scanning.  Exact for any graph.
__global__ void k_defer_filter(const Cont* __restrict__ cand, Act* __restrict__ act,
                               uint8_t* __restrict__ status, uint32_t n, const unsigned long long* __restrict__ Kc) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    if (status[s] != 2) continue;
    const int32_t cv = cand[s].cv;
    const uint32_t kw = (uint32_t)(gat(Kc + cv) >> 32);  // sentinel -> 0xffffffff, never defers
    if (mono_bits(act[s].lb) > kw) {
      status[s] = 4;
      act[s].asleep = 1;
    }
  }
}

// Asleep rows (deferred in an earlier round) are not scanned by pass A at all;
// they only wake when their bound no longer exceeds their component's best
// pass-A offer (or the component has none).  Woken rows are scanned by
// k_offer_warp this round and are awake again if they offer.
__global__ void k_wake(Act* __restrict__ act, uint32_t n, const int32_t* __restrict__ comp,
                       const unsigned long long* __restrict__ Kc, uint8_t* __restrict__ status,
                       Cont* __restrict__ cand) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const int4 r = __ldcs(reinterpret_cast<const int4*>(act + s));
    if (!r.w) continue;
    const int32_t cv = gat(comp + r.x);
    const uint32_t kw = (uint32_t)(gat(Kc + cv) >> 32);
    const bool woken = mono_bits(__int_as_float(r.z)) <= kw;
    status[s] = woken ? 2 : 4;
    if (woken) {
      act[s].asleep = 0;
      __stcs(reinterpret_cast<int4*>(cand + s), make_int4(r.x, r.y, cv, (int)s));
    }
  }
}

__global__ void k_cont_keys(const Cont* __restrict__ c, uint32_t n, int32_t* __restrict__ keys) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) keys[i] = c[i].v;
}


// tie pass over per-slot row offers (status 1)
__global__ void k_tie_slots(const Act* __restrict__ act, const uint8_t* __restrict__ status,
                            const uint64_t* __restrict__ off_key, const uint32_t* __restrict__ off_b, uint32_t n,
                            const int32_t* __restrict__ comp, const uint64_t* __restrict__ Kc,
                            uint32_t* __restrict__ Bc) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    if (status[s] != 1) continue;
    const int32_t c = gat(comp + act[s].v);
    if (off_key[s] == gat(Kc + c)) atomicMin(Bc + c, off_b[s]);
  }
}

// Round 1 with singleton components (exact mode): comp(J) != comp(v) for every
// candidate J, so the first candidate group of the row IS the minimum; no
// component gathers, no atomics, no tie pass -- the owner writes Kc/Bc and the
// hook target directly.
__global__ void k_offer_first(const int32_t* __restrict__ nbr, const float* __restrict__ dist, int32_t k,
                              float eps, int64_t row_begin, int64_t N, const uint32_t* __restrict__ bits,
                              int all_core, const int32_t* __restrict__ comp, Act* __restrict__ act, uint32_t n_in,
                              uint8_t* __restrict__ status, uint64_t* __restrict__ Kc, uint32_t* __restrict__ Bc,
                              int32_t* __restrict__ tgt, unsigned long long* __restrict__ n_entries) {
  unsigned long long reads = 0;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_in; s += gridDim.x * blockDim.x) {
    bool found = false;
    const int32_t v = act[s].v;
    const int64_t i = (int64_t)v - row_begin;
    const int32_t* nr = nbr + i * k;
    const float* dr = dist + i * k;
    uint64_t best = kSent;
    uint32_t bestb = kSentB;
    int64_t bestJ = -1;
    int h = 0;
    float wstar = 0.f;
    for (; h < k; ++h) {
      const float w = __ldcs(dr + h);
      ++reads;
      if (!(w <= eps)) { h = k; break; }
      const int64_t J = __ldcs(nr + h);
      if (!cand_entry(J, v, N, bits, all_core)) continue;
      wstar = w;
      found = true;
      break;
    }
    if (found) {
      for (int h2 = h; h2 < k; ++h2) {
        const float w = h2 == h ? wstar : __ldg(dr + h2);
        if (h2 != h) ++reads;
        if (w != wstar) break;
        const int64_t J = __ldg(nr + h2);
        if (!cand_entry(J, v, N, bits, all_core)) continue;
        const uint64_t kk = pack_key(mono_bits(w), (uint32_t)min((int64_t)v, J));
        const uint32_t bb = (uint32_t)max((int64_t)v, J);
        if (kk < best || (kk == best && bb < bestb)) { best = kk; bestb = bb; bestJ = J; }
      }
      const int32_t cv = gat(comp + v);
      Kc[cv] = best;
      Bc[cv] = bestb;
      tgt[cv] = gat(comp + bestJ);
    }
    act[s].h = min(h, k);
    status[s] = found ? 1 : 0;
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
                           int32_t* __restrict__ off_v, uint64_t* __restrict__ off_key,
                           uint32_t* __restrict__ off_b, uint32_t* __restrict__ n_off,
                           unsigned long long* __restrict__ Kc) {
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
      off_v[o2] = t;
      off_key[o2] = best;
      off_b[o2] = bestb;
      atomicMin(Kc + ct, (unsigned long long)best);
    }
  }
}

// ============================================================================
// a4: tie pass (b of the minimum key)
// ============================================================================
__global__ void k_tie(const int32_t* __restrict__ off_v, const uint64_t* __restrict__ off_key,
                      const uint32_t* __restrict__ off_b, uint32_t n_off,
                      const int32_t* __restrict__ comp, const uint64_t* __restrict__ Kc,
                      uint32_t* __restrict__ Bc) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_off; s += gridDim.x * blockDim.x) {
    const int32_t c = comp[off_v[s]];
    if (off_key[s] == Kc[c]) atomicMin(Bc + c, off_b[s]);
  }
}

// stall fallback (exact mode): offer EVERY live leaving entry of the active
// rows to both endpoint components (rows outside the active list have none)
__global__ void k_sweep(const int32_t* __restrict__ nbr, const float* __restrict__ dist, int32_t k, float eps,
                        int64_t row_begin, int64_t N, const uint32_t* __restrict__ bits,
                        const int32_t* __restrict__ comp, const Act* __restrict__ act, uint32_t n_act,
                        unsigned long long* __restrict__ Kc, uint32_t* __restrict__ Bc, int tie_phase) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_act; s += gridDim.x * blockDim.x) {
    const int64_t v = act[s].v;
    const int64_t i = v - row_begin;
    const int32_t cv = comp[v];
    for (int32_t c = act[s].h; c < k; ++c) {
      const float w = __ldg(dist + i * k + c);
      if (!(w <= eps)) break;
      const int64_t J = __ldg(nbr + i * k + c);
      if (J < 0 || J >= N || J == v || !is_core(bits, J)) continue;
      const int32_t cj = comp[J];
      if (cj == cv) continue;
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

__global__ void k_min_into_u64(uint64_t* __restrict__ d, const uint64_t* __restrict__ s, int64_t n) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    if (s[c] < d[c]) d[c] = s[c];
}
__global__ void k_min_into_u32(uint32_t* __restrict__ d, const uint32_t* __restrict__ s, int64_t n) {
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
__global__ void k_hook(int64_t C, const uint64_t* __restrict__ Kc, const uint32_t* __restrict__ Bc,
                       const int32_t* __restrict__ tgt, const uint32_t* __restrict__ kmin /* null = all certified */,
                       const int32_t* __restrict__ comp, int32_t* __restrict__ parent,
                       uint64_t* __restrict__ e_key, float* __restrict__ e_w, int64_t e_cap,
                       RoundCounters* __restrict__ ctr) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < C;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = base + threadIdx.x;
    bool emit = false, offered = false, unc = false;
    uint32_t a = 0, b = 0, wb = 0;
    if (c < C) {
      const uint64_t K = Kc[c];
      int32_t p = (int32_t)c;
      if (K != kSent) {
        offered = true;
        if (!certified(K, kmin, c)) {
          unc = true;
        } else {
          a = (uint32_t)K;
          b = Bc[c];
          wb = (uint32_t)(K >> 32);
          int32_t t;
          if (tgt) {
            t = tgt[c];
          } else {
            const int32_t x = (gat(comp + a) == (int32_t)c) ? (int32_t)b : (int32_t)a;
            t = gat(comp + x);
          }
          bool mutual, cert_t = true;
          if (kmin) {  // exact mode: t may abstain; also audit the promise
            const uint64_t Kt = gat(Kc + t);
            cert_t = Kt != kSent && certified(Kt, kmin, t);
            // t's true minimum is <= the edge c selected (that edge is incident
            // to t); a larger key means t's offer missed an incident edge --
            // impossible under a true EXACT promise, and the only way a hook
            // cycle longer than a mutual pair could form (Fig. cycle).
            if (cert_t && (Kt > K || (Kt == K && gat(Bc + t) > b))) ctr->violation = 1u;
            mutual = cert_t && Kt == K && gat(Bc + t) == b;
          } else if (tgt) {
            mutual = gat(tgt + t) == (int32_t)c;
          } else {
            mutual = gat(Kc + t) == K && gat(Bc + t) == b;
          }
          if (!(mutual && c < t)) {
            p = t;
            emit = true;
          }
        }
      }
      parent[c] = p;
    }
    block_count(&ctr->offered, offered);
    block_count(&ctr->uncertified, unc);
    block_count(&ctr->hooks, emit);
    const uint32_t slot = block_reserve(&ctr->msf_count, emit);
    if (emit) {
      if ((int64_t)slot < e_cap) {
        e_key[slot] = ((uint64_t)a << 32) | b;
        e_w[slot] = __uint_as_float(wb);
      }
    }
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
__global__ void k_jump(int64_t C, int32_t* parent, int32_t* __restrict__ rootof, RoundCounters* ctr) {
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

__global__ void k_root_flags(int64_t C, const int32_t* __restrict__ rootof, int32_t* __restrict__ flag) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x)
    flag[c] = rootof[c] == (int32_t)c;
}

// new per-component arrays: cmin/kmin are minima over the merged tree
__global__ void k_merge(int64_t C, const int32_t* __restrict__ rootof, const int32_t* __restrict__ newid,
                        const int32_t* __restrict__ cmin, const uint32_t* __restrict__ kmin,
                        int32_t* __restrict__ cmin2, uint32_t* __restrict__ kmin2, int32_t* __restrict__ map) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = gat(newid + rootof[c]);
    map[c] = r;
    atomicMin(cmin2 + r, cmin[c]);
    if (kmin) atomicMin(kmin2 + r, kmin[c]);
  }
}

__global__ void k_fill_i32(int32_t* __restrict__ p, int64_t n, int32_t val) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x)
    p[c] = val;
}

__global__ void k_relabel(int64_t N, int32_t* __restrict__ comp, const int32_t* __restrict__ map) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = comp[v];
    if (c >= 0) comp[v] = gat(map + c);
  }
}

// ============================================================================
// a9 / a11: canonical labels, MSF output, exact weight
// ============================================================================
__global__ void k_canon(int64_t N, int32_t* __restrict__ comp, const int32_t* __restrict__ cmin) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = comp[v];
    if (c >= 0) comp[v] = gat(cmin + c);
  }
}

__global__ void k_split_edges(int64_t m, const uint64_t* __restrict__ keys, uint32_t* __restrict__ a,
                              uint32_t* __restrict__ b) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = keys[e];
    a[e] = (uint32_t)(x >> 32);
    b[e] = (uint32_t)x;
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
__global__ void k_label(const int32_t* __restrict__ nbr, const float* __restrict__ dist, int64_t n_rows,
                        int32_t k, float eps, int64_t row_begin, int64_t N,
                        const uint32_t* __restrict__ bits, const int32_t* __restrict__ comp,
                        int32_t* __restrict__ labels) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = row_begin + i;
    int32_t lab = -1;
    if (is_core(bits, v)) {
      lab = comp[v];
    } else {
      for (int32_t c = 0; c < k; ++c) {
        const float w = __ldg(dist + i * k + c);
        if (!(w <= eps)) break;
        const int64_t J = __ldg(nbr + i * k + c);
        if (J < 0 || J >= N || !is_core(bits, J)) continue;
        lab = comp[J];
        break;
      }
    }
    labels[i] = lab;
  }
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
  Act* act[2] = {nullptr, nullptr};  // active rows (v, head), ping-pong
  Cont* cand = nullptr;               // per-slot continuation records
  Cont* cont = nullptr;               // compacted continuation list
  uint8_t* status = nullptr;          // per slot: 0 exhausted, 1 offer, 2 continue, 4 deferred
  uint32_t n_act = 0;  // live rows in act[cur] (awake and asleep)
  uint32_t n_slots = 0;  // offer slots written by this round's row kernels
  // offers
  int32_t* off_v = nullptr;
  uint64_t* off_key = nullptr;
  uint32_t* off_b = nullptr;
  uint32_t n_off = 0;
  int64_t off_cap_rows = 0;  // offers [0, n_rows) from rows, [n_rows, n_rows + N) from in-lists
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
  uint64_t *e_key, *e_key_sorted;
  float* e_w;
  unsigned long long* buckets;
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
  cub::DeviceRadixSort::SortPairs(nullptr, c, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const float*)nullptr, (float*)nullptr, (int)std::max<int64_t>(cap_edges, 1));
  size_t d = 0, e = 0;
  const int n1 = (int)std::max<int64_t>(N + 1, 1);
  thrust::transform_iterator<IsTwo, const uint8_t*, bool> two(nullptr, IsTwo{});
  cub::DeviceSelect::Flagged(nullptr, d, (const Cont*)nullptr, two, (Cont*)nullptr, (uint32_t*)nullptr, n1);
  cub::DeviceSelect::Flagged(nullptr, e, (const Act*)nullptr, (const uint8_t*)nullptr, (Act*)nullptr,
                             (uint32_t*)nullptr, n1);
  size_t f = 0, g = 0;
  thrust::transform_iterator<IsOne, const uint8_t*, bool> one(nullptr, IsOne{});
  cub::DeviceSelect::Flagged(nullptr, f, (const Act*)nullptr, one, (Act*)nullptr, (uint32_t*)nullptr, n1);
  thrust::transform_iterator<IsFour, const uint8_t*, bool> four(nullptr, IsFour{});
  cub::DeviceSelect::Flagged(nullptr, g, (const Act*)nullptr, four, (Act*)nullptr, (uint32_t*)nullptr, n1);
  f = std::max(f, g);
  size_t h2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, h2, (const int32_t*)nullptr, (int32_t*)nullptr, (const Cont*)nullptr,
                                  (Cont*)nullptr, n1, 0, 32);
  f = std::max(f, h2);
  return std::max(std::max(std::max(a, f), std::max(b, c)), std::max(d, e)) + 256;
}

// carve the workspace; returns bytes needed
size_t carve(Layout& L, char* base, bool dry, int64_t N, int nr, const int64_t* rb, const int64_t* rn,
             bool general, int32_t k) {
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
  L.e_key_sorted = cv.take<uint64_t>(N + 1);
  L.e_w = cv.take<float>(N + 1);
  L.buckets = cv.take<unsigned long long>(256);
  L.ctr = cv.take<RoundCounters>(1);
  L.cub_bytes = cub_tmp_bytes(N, N + 1);
  L.cub_tmp = cv.take<char>(L.cub_bytes);
  L.ranks.assign(nr, RankState());
  for (int r = 0; r < nr; ++r) {
    RankState& R = L.ranks[r];
    R.row_begin = rb[r];
    R.n_rows = rn[r];
    const int64_t n = std::max<int64_t>(rn[r], 1);
    R.act[0] = cv.take<Act>(n);
    R.act[1] = cv.take<Act>(n);
    R.cand = cv.take<Cont>(n);
    R.cont = cv.take<Cont>(n);
    R.status = cv.take<uint8_t>(n);
    const int64_t noff = general ? n + N : n;
    R.off_cap_rows = n;
    R.off_v = cv.take<int32_t>(noff);
    R.off_key = cv.take<uint64_t>(noff);
    R.off_b = cv.take<uint32_t>(noff);
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

kdb_status allreduce_min_u64(kdb_comm* comm, uint64_t* p, int64_t n, cudaStream_t st) {
  if (!comm || comm->kind != 1 || comm->nranks == 1 || n <= 0) return KDB_OK;
  return nccl_check(g_nccl.AllReduce(p, p, (size_t)n, ncclUint64, ncclMin, comm->nccl, st), "ncclAllReduce(u64,min)");
}
kdb_status allreduce_min_u32(kdb_comm* comm, uint32_t* p, int64_t n, cudaStream_t st) {
  if (!comm || comm->kind != 1 || comm->nranks == 1 || n <= 0) return KDB_OK;
  return nccl_check(g_nccl.AllReduce(p, p, (size_t)n, ncclUint32, ncclMin, comm->nccl, st), "ncclAllReduce(u32,min)");
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
  int n = std::min(cap, 8);
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
    LAUNCH(k_core_mark, grid_for(rn[r]), kThreads, st, g->dist + off, rn[r], g->k_max, M, eps, rb[r], core_bits);
    KDB_CUDA(cudaGetLastError());
  }
  // ranks own disjoint bits: SUM == OR
  if (comm && comm->kind == 1 && comm->nranks > 1)
    KDB_TRY(nccl_check(g_nccl.AllReduce(core_bits, core_bits, (size_t)nwords, ncclUint32, ncclSum,
                                        comm->nccl, st), "ncclAllReduce(core bits)"));
  if (g_prof.on) {  // profiling mode only: resolve timings now (synchronises)
    KDB_CUDA(cudaStreamSynchronize(st));
    g_prof.drain();
  }
  return KDB_OK;
}

size_t kdb_mst_workspace_bytes(const kdb_graph* g, kdb_comm* comm) {
  if (validate_graph(g) != KDB_OK) return 0;
  std::vector<int64_t> rb, rn;
  rank_ranges(g, comm, rb, rn);
  Layout L;
  return carve(L, nullptr, true, g->n_total, (int)rb.size(), rb.data(), rn.data(),
               !(g->flags & KDB_GRAPH_EXACT), g->k_max);
}

kdb_status kdb_mst(const kdb_graph* g, float eps, const uint32_t* core_bits, int32_t* comp,
                   uint32_t* mst_a, uint32_t* mst_b, float* mst_w, int64_t mst_cap, int64_t* mst_count,
                   double* mst_weight, void* workspace, size_t ws_bytes, kdb_comm* comm,
                   kdb_stream_t stream) {
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
  const bool general = !(g->flags & KDB_GRAPH_EXACT);
  const int32_t k = g->k_max;
  std::vector<int64_t> rb, rn;
  rank_ranges(g, comm, rb, rn);
  Layout L;
  const size_t need = carve(L, (char*)workspace, false, N, (int)rb.size(), rb.data(), rn.data(), general, k);
  if (ws_bytes < need) return set_err(KDB_ENOMEM, "workspace %zu < required %zu bytes", ws_bytes, need);
  *mst_count = 0;
  *mst_weight = 0.0;
  for (auto& s : g_stats) s = 0;
  if (N == 0) return KDB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  for (auto& R : L.ranks) {
    R.nbr = g->nbr + (R.row_begin - g->row_begin) * k;
    R.dist = g->dist + (R.row_begin - g->row_begin) * k;
  }
  cudaEvent_t ev[4];
  for (auto& e : ev) KDB_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() { for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]); }
  } guard{ev};
  float ms = 0;
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
  L.all_core = (C == N) ? 1 : 0;  // then no entry needs a core-bit gather
  LAUNCH(k_init_comp, grid_for(N), kThreads, st, core_bits, L.woff, N, comp, L.cmin);
  LAUNCH(k_fill_comp_arrays, grid_for(C), kThreads, st, C, L.Kc, L.Bc, general ? nullptr : L.kmin);
  for (size_t r = 1; r < L.ranks.size(); ++r)
    LAUNCH(k_fill_comp_arrays, grid_for(C), kThreads, st, C, L.ranks[r].Kc, L.ranks[r].Bc, nullptr);
  KDB_CUDA(cudaGetLastError());
  for (auto& R : L.ranks) {
    KDB_CUDA(cudaMemsetAsync(R.ctr, 0, sizeof(RoundCounters), st));
    if (R.n_rows > 0) {
      // every row as (v, 0) + a flag, then a stable select: the active list is in row order
      LAUNCH(k_init_rows, grid_for(R.n_rows), kThreads, st, R.dist, R.n_rows, k, eps, R.row_begin, core_bits, comp,
             general ? nullptr : L.kmin, R.act[1], R.status);
      cb = L.cub_bytes;
      { LaunchScope ls_("cub::DeviceSelect", st, false);
        KDB_CUDA(cub::DeviceSelect::Flagged(L.cub_tmp, cb, R.act[1], R.status, R.act[0], &R.ctr->n_act[0],
                                            (int)R.n_rows, st)); }
    }
    KDB_CUDA(cudaGetLastError());
  }
  if (!general) {
    KDB_TRY(allreduce_min_u32(comm, L.kmin, C, st));
    for (auto& R : L.ranks) LAUNCH(k_fill_i32, grid_for(C), kThreads, st, R.tgt, C, INT32_MAX);
  }
  KDB_CUDA(cudaEventRecord(ev[1], st));
  // ---- general mode: in-edge lists --------------------------------------------
  if (general) {
    for (auto& R : L.ranks) {
      // counts -> scan -> offsets; e_key (N+1 u64) is scratch for counts and cursors
      unsigned long long* cursor = reinterpret_cast<unsigned long long*>(L.e_key);
      KDB_CUDA(cudaMemsetAsync(cursor, 0, (N + 1) * sizeof(unsigned long long), st));
      if (R.n_rows > 0)
        LAUNCH(k_in_count, grid_for(R.n_rows), kThreads, st, R.nbr, R.dist, R.n_rows, k, eps, R.row_begin, N,
                                                            core_bits, cursor);
      cb = L.cub_bytes;
      { LaunchScope ls_("cub::DeviceScan", st, false); KDB_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb, cursor, R.in_off, (int)(N + 1), st)); }
      KDB_CUDA(cudaMemcpyAsync(cursor, R.in_off, (N + 1) * sizeof(unsigned long long),
                               cudaMemcpyDeviceToDevice, st));
      if (R.n_rows > 0)
        LAUNCH(k_in_fill, grid_for(R.n_rows), kThreads, st, R.nbr, R.dist, R.n_rows, k, eps, R.row_begin, N,
                                                           core_bits, cursor, R.in_src, R.in_w);
      LAUNCH(k_in_finish, grid_for(N), kThreads, st, R.in_off, N, R.in_len, R.in_act[0], &R.ctr->n_act[1]);
      KDB_CUDA(cudaGetLastError());
    }
  }
  for (auto& R : L.ranks) {
    RoundCounters hc;
    KDB_CUDA(cudaMemcpyAsync(&hc, R.ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    R.n_act = hc.n_act[0];  // initial active rows are all awake
    R.n_in_act = hc.n_act[1];
  }
  KDB_CUDA(cudaEventRecord(ev[2], st));
  KDB_CUDA(cudaEventSynchronize(ev[2]));
  KDB_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
  g_stats[1] = ms;
  KDB_CUDA(cudaEventElapsedTime(&ms, ev[1], ev[2]));
  g_stats[5] = ms;

  // ---- Boruvka rounds -------------------------------------------------------------
  int cur = 0;
  int rounds = 0, stalls = 0;
  const uint32_t* kmin_cert = general ? nullptr : L.kmin;
  double t_min_edges = 0, t_contract = 0;
  while (C > 0) {
    ++rounds;
    // round 1 of exact mode: singleton components, one offer each (no in-lists)
    const bool direct = rounds == 1 && !general;
    KDB_CUDA(cudaEventRecord(ev[0], st));
    // a3: offers (rows, then in-lists), per rank, into that rank's Kc partial
    for (auto& R : L.ranks) {
      KDB_CUDA(cudaMemsetAsync(&R.ctr->n_act[0], 0, 3 * sizeof(uint32_t), st));  // n_act[0..1], n_off
      R.n_slots = 0;
      // one list of live rows in row order; a flag in each record marks asleep rows
      const uint32_t n_in = R.n_act;
      if (n_in) {
        if (direct) {
          LAUNCH(k_offer_first, grid_for(n_in), kThreads, st, R.nbr, R.dist, k, eps, R.row_begin, N, core_bits,
                 L.all_core, comp, R.act[cur], n_in, R.status, R.Kc, R.Bc, R.tgt, &L.ctr->entries);
        } else {
          // pass A: the first chunk of every awake row
          for (uint32_t s0 = 0; s0 < n_in; s0 += g_chunk) {
            const uint32_t s1 = std::min<uint32_t>(s0 + g_chunk, n_in);
            if ((k % 4) == 0)
              LAUNCH(k_offer_rows_t<true>, grid_for(s1 - s0), kThreads, st, R.nbr, R.dist, k, eps, R.row_begin, N,
                     core_bits, L.all_core, comp, R.act[cur], s0, s1, R.status, R.off_key, R.off_b, nullptr,
                     (unsigned long long*)R.Kc, &L.ctr->entries, g_qmax);
            else
              LAUNCH(k_offer_rows_t<false>, grid_for(s1 - s0), kThreads, st, R.nbr, R.dist, k, eps, R.row_begin, N,
                     core_bits, L.all_core, comp, R.act[cur], s0, s1, R.status, R.off_key, R.off_b, nullptr,
                     (unsigned long long*)R.Kc, &L.ctr->entries, g_qmax);
          }
          // lazy Boruvka + scans of the rows that might supply their component's minimum
          KDB_CUDA(cudaMemsetAsync(&R.ctr->n_cont, 0, sizeof(uint32_t), st));
          LAUNCH(k_scan_tiles, grid_for((int64_t)n_in), kThreads, st, R.nbr, R.dist, k, eps, R.row_begin, N,
                 core_bits, L.all_core, comp, R.act[cur], n_in, R.status, R.off_key, R.off_b,
                 (unsigned long long*)R.Kc, g_lazy, &L.ctr->entries, &R.ctr->n_cont, g_fa, g_fs);
        }
        // next list: rows that offered (awake) or were deferred (asleep), row order kept
        cb = L.cub_bytes;
        {
          LaunchScope ls_("cub::DeviceSelect", st, false);
          thrust::transform_iterator<Survives, const uint8_t*, bool> keep(R.status, Survives{});
          KDB_CUDA(cub::DeviceSelect::Flagged(L.cub_tmp, cb, R.act[cur], keep, R.act[cur ^ 1], &R.ctr->n_act[0],
                                              (int)n_in, st));
        }
        R.n_slots = direct ? 0 : n_in;
      }
      if (general && R.n_in_act)
        LAUNCH(k_offer_in, grid_for(R.n_in_act), kThreads, st, R.in_off, R.in_len, R.in_src, R.in_w, comp,
               R.in_act[cur], R.n_in_act, R.in_act[cur ^ 1], &R.ctr->n_act[1], R.off_v + R.off_cap_rows,
               R.off_key + R.off_cap_rows, R.off_b + R.off_cap_rows, &R.ctr->n_off, (unsigned long long*)R.Kc);
      KDB_CUDA(cudaGetLastError());
    }
    if (g_trace) {
      RoundCounters h0, hr;
      KDB_CUDA(cudaMemcpyAsync(&h0, L.ctr, sizeof(h0), cudaMemcpyDeviceToHost, st));
      KDB_CUDA(cudaMemcpyAsync(&hr, L.ranks[0].ctr, sizeof(hr), cudaMemcpyDeviceToHost, st));
      KDB_CUDA(cudaEventRecord(ev[3], st));
      KDB_CUDA(cudaEventSynchronize(ev[3]));
      float tms = 0;
      KDB_CUDA(cudaEventElapsedTime(&tms, ev[0], ev[3]));
      static unsigned long long last_entries = 0;
      if (rounds == 1) last_entries = 0;
      fprintf(stderr, "[kdb] round %d C=%lld live=%u scanned=%u -> live=%u entries=%llu offer_ms=%.3f\n",
              rounds, (long long)C, L.ranks[0].n_act, hr.n_cont, hr.n_act[0], h0.entries - last_entries, tms);
      last_entries = h0.entries;
    }
    for (auto& R : L.ranks) {
      RoundCounters hc;
      KDB_CUDA(cudaMemcpyAsync(&hc, R.ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
      KDB_CUDA(cudaStreamSynchronize(st));
      R.n_act = hc.n_act[0];
      R.n_in_act = hc.n_act[1];
      R.n_off = hc.n_off;  // in-list offers (row offers live in the row slots)
    }
    // exchange: sim -> min over virtual ranks; nccl -> allreduce
    for (size_t r = 1; r < L.ranks.size(); ++r)
      LAUNCH(k_min_into_u64, grid_for(C), kThreads, st, L.Kc, L.ranks[r].Kc, C);
    KDB_TRY(allreduce_min_u64(comm, L.Kc, C, st));
    // a4: ties (the direct round already wrote Bc and the targets)
    for (auto& R : L.ranks) {
      if (R.n_slots && !direct)
        LAUNCH(k_tie_slots, grid_for(R.n_slots), kThreads, st, R.act[cur], R.status, R.off_key, R.off_b,
               R.n_slots, comp, L.Kc, R.Bc);
      if (R.n_off && !direct)
        LAUNCH(k_tie, grid_for(R.n_off), kThreads, st, R.off_v + R.off_cap_rows, R.off_key + R.off_cap_rows,
               R.off_b + R.off_cap_rows, R.n_off, comp, L.Kc, R.Bc);
      KDB_CUDA(cudaGetLastError());
    }
    for (size_t r = 1; r < L.ranks.size(); ++r)
      LAUNCH(k_min_into_u32, grid_for(C), kThreads, st, L.Bc, L.ranks[r].Bc, C);
    KDB_TRY(allreduce_min_u32(comm, L.Bc, C, st));
    if (direct) {
      for (size_t r = 1; r < L.ranks.size(); ++r)
        LAUNCH(k_min_into_u32, grid_for(C), kThreads, st, (uint32_t*)L.tgt, (const uint32_t*)L.ranks[r].tgt, C);
      KDB_TRY(allreduce_min_u32(comm, (uint32_t*)L.tgt, C, st));  // non-owners hold INT32_MAX
    }
    KDB_CUDA(cudaEventRecord(ev[1], st));
    // a5: hook + emit
    KDB_CUDA(cudaMemsetAsync(&L.ctr->hooks, 0, 4 * sizeof(uint32_t), st));
    LAUNCH(k_hook, grid_for(C), kThreads, st, C, L.Kc, L.Bc, direct ? L.tgt : nullptr, kmin_cert, comp, L.parent,
           L.e_key, L.e_w, N, L.ctr);
    KDB_CUDA(cudaGetLastError());
    RoundCounters hc;
    KDB_CUDA(cudaMemcpyAsync(&hc, L.ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    if (hc.offered == 0) {  // a8: no component has a leaving edge
      KDB_CUDA(cudaEventRecord(ev[2], st));
      KDB_CUDA(cudaEventSynchronize(ev[2]));
      KDB_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
      t_min_edges += ms;
      break;
    }
    if (hc.hooks == 0) {
      // every offering component abstained: one edge-centric sweep round gives
      // every component its exact minimum (both endpoints see every entry)
      ++stalls;
      LAUNCH(k_fill_comp_arrays, grid_for(C), kThreads, st, C, L.Kc, L.Bc, nullptr);
      for (size_t r = 1; r < L.ranks.size(); ++r)
        LAUNCH(k_fill_comp_arrays, grid_for(C), kThreads, st, C, L.ranks[r].Kc, L.ranks[r].Bc, nullptr);
      for (auto& R : L.ranks)
        if (R.n_rows)
          LAUNCH(k_sweep, grid_for(R.n_act), kThreads, st, R.nbr, R.dist, k, eps, R.row_begin, N, core_bits,
                 comp, R.act[cur ^ 1], R.n_act, (unsigned long long*)R.Kc, R.Bc, 0);
      for (size_t r = 1; r < L.ranks.size(); ++r)
        LAUNCH(k_min_into_u64, grid_for(C), kThreads, st, L.Kc, L.ranks[r].Kc, C);
      KDB_TRY(allreduce_min_u64(comm, L.Kc, C, st));
      for (auto& R : L.ranks)
        if (R.n_rows)
          LAUNCH(k_sweep, grid_for(R.n_act), kThreads, st, R.nbr, R.dist, k, eps, R.row_begin, N, core_bits,
                 comp, R.act[cur ^ 1], R.n_act, (unsigned long long*)L.Kc, R.Bc, 1);
      for (size_t r = 1; r < L.ranks.size(); ++r)
        LAUNCH(k_min_into_u32, grid_for(C), kThreads, st, L.Bc, L.ranks[r].Bc, C);
      KDB_TRY(allreduce_min_u32(comm, L.Bc, C, st));
      KDB_CUDA(cudaMemsetAsync(&L.ctr->hooks, 0, 4 * sizeof(uint32_t), st));
      LAUNCH(k_hook, grid_for(C), kThreads, st, C, L.Kc, L.Bc, nullptr, nullptr, comp, L.parent, L.e_key, L.e_w, N,
                                               L.ctr);
      KDB_CUDA(cudaGetLastError());
      KDB_CUDA(cudaMemcpyAsync(&hc, L.ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
      KDB_CUDA(cudaStreamSynchronize(st));
      if (hc.hooks == 0) return set_err(KDB_EINTERNAL, "sweep round made no progress");
      // vertices whose rows were exhausted stay out of the active list; rows
      // that still hold leaving entries are in it (exhaustion is permanent)
    }
    if (hc.violation) return set_err(KDB_EINVAL, "graph violates the KDB_GRAPH_EXACT promise (a component's "
                                     "minimum missed an incident edge)");
    // a6: contract
    LAUNCH(k_jump, grid_for(C), kThreads, st, C, L.parent, L.rootof, L.ctr);
    LAUNCH(k_root_flags, grid_for(C), kThreads, st, C, L.rootof, L.flag);
    cb = L.cub_bytes;
    { LaunchScope ls_("cub::DeviceScan", st, false); KDB_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb, L.flag, L.newid, (int)C, st)); }
    uint32_t viol = 0;
    KDB_CUDA(cudaMemcpyAsync(&viol, &L.ctr->violation, 4, cudaMemcpyDeviceToHost, st));
    int32_t last[2];
    KDB_CUDA(cudaMemcpyAsync(&last[0], L.newid + C - 1, 4, cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaMemcpyAsync(&last[1], L.flag + C - 1, 4, cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    if (viol) return set_err(KDB_EINTERNAL, "pointer jumping did not converge (hook cycle)");
    const int64_t C2 = (int64_t)last[0] + last[1];
    LAUNCH(k_fill_i32, grid_for(C2), kThreads, st, L.cmin2, C2, INT32_MAX);
    if (!general) LAUNCH(k_fill_i32, grid_for(C2), kThreads, st, (int32_t*)L.kmin2, C2, (int32_t)kInfBits);
    // map[c] = new dense id of c's tree (reuses `parent`, no longer needed)
    LAUNCH(k_merge, grid_for(C), kThreads, st, C, L.rootof, L.newid, L.cmin, general ? nullptr : L.kmin, L.cmin2,
           L.kmin2, L.parent);
    LAUNCH(k_relabel, grid_for(N), kThreads, st, N, comp, L.parent);
    LAUNCH(k_fill_comp_arrays, grid_for(C2), kThreads, st, C2, L.Kc, L.Bc, nullptr);
    for (size_t r = 1; r < L.ranks.size(); ++r)
      LAUNCH(k_fill_comp_arrays, grid_for(C2), kThreads, st, C2, L.ranks[r].Kc, L.ranks[r].Bc, nullptr);
    KDB_CUDA(cudaGetLastError());
    std::swap(L.cmin, L.cmin2);
    std::swap(L.kmin, L.kmin2);
    kmin_cert = general ? nullptr : L.kmin;
    C = C2;
    cur ^= 1;
    KDB_CUDA(cudaEventRecord(ev[2], st));
    KDB_CUDA(cudaEventSynchronize(ev[2]));
    KDB_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    t_min_edges += ms;
    KDB_CUDA(cudaEventElapsedTime(&ms, ev[1], ev[2]));
    t_contract += ms;
  }
  // ---- finalize ---------------------------------------------------------------------
  KDB_CUDA(cudaEventRecord(ev[0], st));
  RoundCounters hc;
  KDB_CUDA(cudaMemcpyAsync(&hc, L.ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
  KDB_CUDA(cudaStreamSynchronize(st));
  const int64_t m = (int64_t)hc.msf_count;
  if (m > N) return set_err(KDB_EINTERNAL, "MSF larger than N-1");
  if (m > mst_cap) return set_err(KDB_EINVAL, "mst_cap %lld < MSF size %lld", (long long)mst_cap, (long long)m);
  LAUNCH(k_canon, grid_for(N), kThreads, st, N, comp, L.cmin);
  KDB_CUDA(cudaGetLastError());
  unsigned long long bk[256];
  if (m > 0) {
    cb = L.cub_bytes;
    { LaunchScope ls_("cub::DeviceRadixSort", st, false); KDB_CUDA(cub::DeviceRadixSort::SortPairs(L.cub_tmp, cb, L.e_key, L.e_key_sorted, L.e_w, mst_w, (int)m, 0, 64, st)); }
    LAUNCH(k_split_edges, grid_for(m), kThreads, st, m, L.e_key_sorted, mst_a, mst_b);
    KDB_CUDA(cudaMemsetAsync(L.buckets, 0, 256 * sizeof(unsigned long long), st));
    LAUNCH(k_wbuckets, grid_for(m), kThreads, st, m, mst_w, L.buckets);
    KDB_CUDA(cudaGetLastError());
    KDB_CUDA(cudaMemcpyAsync(bk, L.buckets, sizeof(bk), cudaMemcpyDeviceToHost, st));
  }
  KDB_CUDA(cudaEventRecord(ev[1], st));
  KDB_CUDA(cudaStreamSynchronize(st));
  KDB_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
  if (g_prof.on) g_prof.drain();
  *mst_count = m;
  *mst_weight = m > 0 ? exact_bucket_sum(bk) : 0.0;
  g_stats[0] = rounds;
  g_stats[2] = t_min_edges;
  g_stats[3] = t_contract;
  g_stats[4] = ms;
  g_stats[6] = stalls;
  g_stats[7] = (double)hc.entries;
  return KDB_OK;
}

kdb_status kdb_label(const kdb_graph* g, float eps, const uint32_t* core_bits, const int32_t* comp,
                     int32_t* labels, kdb_stream_t stream) {
  KDB_TRY(validate_graph(g));
  KDB_TRY(validate_eps(eps));
  if (g->n_rows > 0 && (!core_bits || !comp || !labels)) return set_err(KDB_EINVAL, "NULL device pointer");
  if (g->n_rows == 0) return KDB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  LAUNCH(k_label, grid_for(g->n_rows), kThreads, st, g->nbr, g->dist, g->n_rows, g->k_max, eps, g->row_begin,
                                                    g->n_total, core_bits, comp, labels);
  KDB_CUDA(cudaGetLastError());
  if (g_prof.on) {
    KDB_CUDA(cudaStreamSynchronize(st));
    g_prof.drain();
  }
  return KDB_OK;
}

}  // extern "C"
