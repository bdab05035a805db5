// kdb.cu -- B200-native (sm_100a) kNN-DBSCAN clustering stage behind the C-ABI
// declared in include/kdb.h.  One translation unit: this file (helpers,
// profiling, NCCL loader, the C-ABI entry points, NMI) includes kdb_rows.cuh
// (a1-a11 round kernels), kdb_filter.cuh (Filter-Boruvka and inexact-MST
// kernels) and kdb_host.cuh (workspace layout and the phases).
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
#include <cub/device/device_segmented_sort.cuh>
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
#include <mutex>
#include <string>
#include <vector>

// ============================================================================
// error plumbing
// ============================================================================
namespace {

thread_local std::string g_err;
thread_local double g_stats[32];

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

#ifndef KDB_GUARDS
#define KDB_GUARDS 0
#endif
constexpr size_t kGuardBytes = KDB_GUARDS ? 256 : 0;
constexpr unsigned char kGuardByte = 0xA5;
// debug build: device-side bounds checks record a bit here instead of trapping
__device__ unsigned int g_dbg_viol = 0;
#if KDB_GUARDS
#define KDB_DCHECK(cond, bit) \
  do {                        \
    if (!(cond)) atomicOr(&g_dbg_viol, (bit)); \
  } while (0)
#else
#define KDB_DCHECK(cond, bit) \
  do {                        \
  } while (0)
#endif

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
// CTAs per SM x SMs), from the occupancy calculator (cached per device, kernel,
// block size and dynamic shared memory; the cache is shared by host threads).
// A second wave would only start after the first finished ALL its strides.
struct CapKey {
  int dev;
  const void* kern;
  int block;
  size_t smem;
};
std::mutex g_cap_mu;
std::vector<std::pair<CapKey, int>> g_cap_cache;
int resident_cap_smem(const void* kern, int block, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cap_mu);
  for (auto& e : g_cap_cache)
    if (e.first.dev == dev && e.first.kern == kern && e.first.block == block && e.first.smem == smem)
      return e.second;
  // dynamic shared memory above 48 KB needs the opt-in on THIS device
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms = 0, per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  g_cap_cache.push_back({CapKey{dev, kern, block, smem}, per_sm * sms});
  return per_sm * sms;
}
int resident_cap(const void* kern, int block) { return resident_cap_smem(kern, block, 0); }

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
// ============================================================================
// Tuning options (experiment switches): set only through
// kdb_set_option (include/kdb.h); the library never reads them from the
// environment.  Every call site names its own default, which is what runs
// unless the caller overrode the option.
// ============================================================================
const char* const kOptNames[] = {
    "KDB_CAS",      "KDB_COMPACT", "KDB_FASTFILTER", "KDB_FASTSCAN", "KDB_FILTER",  "KDB_FUSE1",   "KDB_GM",  "KDB_GMAP",      "KDB_GW",
    "KDB_L1GAT",    "KDB_L2HINT",  "KDB_LEAN",       "KDB_LIGHT",   "KDB_LOCAL",   "KDB_LVL",  "KDB_MSF_COUNT", "KDB_NCCL_FORCE",
    "KDB_PACK1",    "KDB_PIPE",    "KDB_PIPE_R0",    "KDB_PIPE_R1", "KDB_PRECHECK", "KDB_QUAD", "KDB_REFILL", "KDB_REUSE",    "KDB_SKIP1",
    "KDB_SPARSE",   "KDB_SURVCAP", "KDB_TILE",       "KDB_TILE_MAXR", "KDB_TILE_ROWS", "KDB_TRACE"};
constexpr int kNumOpts = (int)(sizeof(kOptNames) / sizeof(kOptNames[0]));
std::mutex g_opt_mu;
long long g_opt_val[kNumOpts];
bool g_opt_isset[kNumOpts];
int opt_index(const char* name) {
  if (!name) return -1;
  for (int i = 0; i < kNumOpts; ++i)
    if (strcmp(kOptNames[i], name) == 0) return i;
  return -1;
}
// the caller's value of option `name`, else the call site's default
int opt_int(const char* name, int dflt) {
  const int i = opt_index(name);
  std::lock_guard<std::mutex> lk(g_opt_mu);
  return (i >= 0 && g_opt_isset[i]) ? (int)g_opt_val[i] : dflt;
}
bool opt_set(const char* name) {
  const int i = opt_index(name);
  std::lock_guard<std::mutex> lk(g_opt_mu);
  return i >= 0 && g_opt_isset[i];
}
bool trace_on() { return opt_int("KDB_TRACE", 0) != 0; }  // per-round log to stderr

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
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
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
  g_nccl.Broadcast = (decltype(g_nccl.Broadcast))dlsym(h, "ncclBroadcast");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
  g_nccl.GroupStart = (decltype(g_nccl.GroupStart))dlsym(h, "ncclGroupStart");
  g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))dlsym(h, "ncclGroupEnd");
  if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.AllReduce || !g_nccl.CommDestroy ||
      !g_nccl.Broadcast || !g_nccl.AllGather || !g_nccl.GroupStart || !g_nccl.GroupEnd)
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

// 128-bit compare-and-swap minimum of the pair (key, b) (sm_90+ atom.cas.b128):
// the full O1 order in one atomic word, so one rank needs no separate tie pass
// and no offer list.  A torn 128-bit read only makes the first CAS fail; the
// CAS returns the true current pair and the loop re-tests against it.
__device__ __forceinline__ ulonglong2 atom_cas128(ulonglong2* p, ulonglong2 cmp, ulonglong2 val) {
  ulonglong2 old;
  asm volatile(
      "{\n\t.reg .b128 d, c, v;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 v, {%4, %5};\n\t"
      "atom.global.cas.b128 d, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(old.x), "=l"(old.y)
      : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(p)
      : "memory");
  return old;
}
__device__ __forceinline__ void min_pair128(ulonglong2* p, uint64_t key, uint64_t b) {
  ulonglong2 cur = __ldcg(p);
  while (key < cur.x || (key == cur.x && b < cur.y)) {
    const ulonglong2 old = atom_cas128(p, cur, make_ulonglong2(key, b));
    if (old.x == cur.x && old.y == cur.y) break;
    cur = old;
  }
}

// Warp-collective min_pair128: lanes offering to the SAME component in a run
// of consecutive lanes (rows of one component next to each other in the row
// order, e.g. spatially ordered ids) are min-reduced first and only the run's
// first lane issues the CAS -- same-address CAS loops serialise at the L2
// slice.  A warp with no such run (random ids) pays one shuffle and a ballot.
// Lanes with have == false must pass a c that no other lane holds.
__device__ __forceinline__ void warp_min_pair128(ulonglong2* KB, bool have, int32_t c, uint64_t key, uint64_t b) {
  const int lane = threadIdx.x & 31;
  const int32_t cn = __shfl_down_sync(0xffffffffu, c, 1);
  const unsigned last = __ballot_sync(0xffffffffu, lane == 31 || cn != c);  // lane ends its run
  if (last != 0xffffffffu) {
    const int end = lane + __ffs(last >> lane) - 1;
    const unsigned longest = __reduce_max_sync(0xffffffffu, (unsigned)(end - lane + 1));  // warp-uniform
    for (int o = 1; o < (int)longest; o <<= 1) {
      const uint64_t ok = __shfl_down_sync(0xffffffffu, key, o);
      const uint64_t obb = __shfl_down_sync(0xffffffffu, b, o);
      if (lane + o <= end && (ok < key || (ok == key && obb < b))) { key = ok; b = obb; }
    }
    const int32_t cp = __shfl_up_sync(0xffffffffu, c, 1);
    if (lane > 0 && cp == c) have = false;  // not the first lane of its run
  }
  if (have) min_pair128(KB + c, key, b);
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
  uint32_t n_deep;               // per rank: rows whose kW ELL entries are all within eps_run
  uint32_t n_local;              // per rank: rows whose nearest neighbour's id is within 2^16 of
                                 // their own (spatially ordered ids: the component gathers go through L1)
  uint32_t grab;                 // chunk cursor of the ordered row kernels (per rank)
  uint32_t n_off2;
  uint32_t n_park;               // per rank, local-first phase: rows parked for the global phase
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


#include "kdb_rows.cuh"
#include "kdb_tile.cuh"
#include "kdb_filter.cuh"
#include "kdb_host.cuh"

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

kdb_status kdb_set_option(const char* name, long long value) {
  const int i = opt_index(name);
  if (i < 0) return set_err(KDB_EINVAL, "unknown option '%s'", name ? name : "(null)");
  std::lock_guard<std::mutex> lk(g_opt_mu);
  g_opt_val[i] = value;
  g_opt_isset[i] = true;
  return KDB_OK;
}

int kdb_get_option(const char* name, long long* value) {
  const int i = opt_index(name);
  if (i < 0) return -1;
  std::lock_guard<std::mutex> lk(g_opt_mu);
  if (value) *value = g_opt_isset[i] ? g_opt_val[i] : 0;
  return g_opt_isset[i] ? 1 : 0;
}

void kdb_reset_options(void) {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  for (int i = 0; i < kNumOpts; ++i) g_opt_isset[i] = false;
}

int kdb_option_name(int i, const char** name) {
  if (i < 0 || i >= kNumOpts) return 0;
  if (name) *name = kOptNames[i];
  return 1;
}

int kdb_last_mst_stats(double* out, int cap) {
  int n = std::min(cap, 32);
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
               edge_cols_of(g), -1, local_first_on(g, comm));
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
  // whatever this call does, a kept light ELL in this workspace is not valid
  // after it unless this call keeps a new one (see EllKey)
  const void* ws0 = workspace;
  EllKey ell_prev = ell_take(ws0);
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
  m.lf = !inexact && !m.general && local_first_on(g, comm);
  // a kept light ELL is only valid until the workspace's next call: take it out
  // of the table now, put a new one back on success
  m.ws = ws0;
  m.reuse_req = (g->flags & KDB_GRAPH_REUSE) != 0 && opt_int("KDB_REUSE", 1) != 0;
  m.ell_prev = ell_prev;
  Layout& L = m.L;
  std::vector<int64_t> rb, rn;
  rank_ranges(g, comm, rb, rn);
  const size_t need = carve(L, (char*)workspace, false, N, (int)rb.size(), rb.data(), rn.data(), m.general, m.k,
                            inexact ? g->n_rows * (int64_t)m.k : -1, local_first_on(g, comm) && !inexact);
  if (ws_bytes < need) return set_err(KDB_ENOMEM, "workspace %zu < required %zu bytes", ws_bytes, need);
  KDB_TRY(guards_fill((char*)workspace, L.guards, (cudaStream_t)stream));
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
  const int light_m = opt_int("KDB_LIGHT", 10);
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
    uint32_t nc[2] = {0, 0};  // count, sticky overflow flag
    KDB_CUDA(cudaMemcpyAsync(nc, R.n_hs_dev, 8, cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    const uint32_t ncut = nc[0];
    if (ncut > R.hs_cap || nc[1]) return set_err(KDB_EINTERNAL, "cut entries exceed their buffer");
    R.n_hs = ncut;
    m.survivors = ncut;
    KDB_CUDA(cudaEventRecord(m.ev[1], st));
    m.t_filter += elapsed(m.ev[0], m.ev[1]);
    KDB_TRY(heavy_phase(m));
  } else if (opt_int("KDB_FILTER", 1) && light_m >= 1 && light_m < m.k &&
             (opt_set("KDB_LIGHT") || m.k >= 4 * light_m)) {
    // default policy: split only when the rows are long next to the light
    // prefix (k >= 4 x the light column): with k = 16 / 32 the filter pass and
    // the heavy phase cost more than the rows phase saves (C1 1.49 -> 0.99 ms,
    // C2 3.69 -> 2.27 ms without the split; C3 / C4 (k = 100) gain from it).
    // An explicit KDB_LIGHT always splits (tests, tuning).
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
  int64_t ne = (int64_t)hc.msf_count;
  if (ne > N) return set_err(KDB_EINTERNAL, "MSF larger than N-1");
  const bool dist_out = multi_rank(comm);
  if (dist_out && ne > 0) {
    // multi-rank output (kdb.h): this rank returns the MSF edges whose smaller
    // endpoint lies in its rows -- its local-phase edges and its share of the
    // replicated global / heavy-phase edges
    RankState& R0 = L.ranks[0];
    KDB_CUDA(cudaMemsetAsync(&L.ctr->n_off, 0, sizeof(uint32_t), st));
    LAUNCH(k_keep_a_range, grid_for(ne), kThreads, st, L.e_key, reinterpret_cast<const uint32_t*>(L.e_w), ne,
           R0.row_begin, R0.row_begin + R0.n_rows, L.Kc, L.Bc, &L.ctr->n_off);
    KDB_CUDA(cudaGetLastError());
    uint32_t kept = 0;
    KDB_CUDA(cudaMemcpyAsync(&kept, &L.ctr->n_off, sizeof(kept), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    std::swap(L.e_key, L.Kc);
    float* w = L.e_w;
    L.e_w = reinterpret_cast<float*>(L.Bc);
    L.Bc = reinterpret_cast<uint32_t*>(w);
    ne = kept;
  }
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
    if (4 * ne >= N && opt_int("KDB_MSF_COUNT", 0) != 0) {
      // dense forest (C4: N - 10 edges): a counting sort by a over the N ids --
      // one atomic and one scatter per edge instead of the radix sort's passes.
      // Off by default (KDB_MSF_COUNT=1): C4 2.0 ms (scatter 1.41, count 0.47,
      // scan 0.14) against the radix sort's 2.08 ms -- the random 12-B scatter
      // costs what the passes save
      uint32_t* cnt = reinterpret_cast<uint32_t*>(L.flag);     // N + 1, free after the phases
      uint32_t* off = reinterpret_cast<uint32_t*>(L.rootof);   // N + 1
      uint32_t* pos = reinterpret_cast<uint32_t*>(L.tgt);      // N + 1 >= ne
      const uint32_t* ea = reinterpret_cast<const uint32_t*>(L.e_w);
      KDB_CUDA(cudaMemsetAsync(cnt, 0, (N + 1) * sizeof(uint32_t), st));
      LAUNCH(k_msf_count, grid_for(ne), kThreads, st, ne, ea, cnt, pos);
      { LaunchScope ls_("cub::DeviceScan", st, false);
        KDB_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb, cnt, off, (int)(N + 1), st)); }
      LAUNCH(k_msf_scatter, grid_for(ne), kThreads, st, ne, ea, reinterpret_cast<const unsigned long long*>(L.e_key),
             off, pos, reinterpret_cast<uint32_t*>(mst_a), vb2);
      KDB_CUDA(cudaGetLastError());
    } else {
      // the emitted (a, (b, w)) pairs sort straight into the caller's mst_a
      LaunchScope ls_("cub::DeviceRadixSort", st, false);
      KDB_CUDA(cub::DeviceRadixSort::SortPairs(L.cub_tmp, cb, reinterpret_cast<const uint32_t*>(L.e_w), mst_a,
                                               reinterpret_cast<const unsigned long long*>(L.e_key), vb2, (int)ne, 0,
                                               abits, st));
    }
    // runs of equal a longer than kRunMax (a hub vertex: duplicates, stars) are
    // left to a segmented sort instead of one thread's insertion sort
    int32_t* seg_b = L.cmin2;  // free after the phases
    int32_t* seg_e = L.newid;
    KDB_CUDA(cudaMemsetAsync(&L.ctr->n_off, 0, sizeof(uint32_t), st));
    LAUNCH(k_msf_unpack, grid_for(ne), kThreads, st, ne, mst_a, vb2, mst_b, mst_w, seg_b, seg_e, &L.ctr->n_off);
    uint32_t nseg = 0;
    KDB_CUDA(cudaMemcpyAsync(&nseg, &L.ctr->n_off, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    if (nseg > 0) {
      uint32_t* kout = reinterpret_cast<uint32_t*>(vb2);  // vb2 (8 (N + 1) bytes) is free after the unpack
      float* vout = reinterpret_cast<float*>(kout + ne);
      size_t cbs = L.cub_bytes;
      {
        LaunchScope ls_("cub::DeviceSegmentedSort", st, false);
        KDB_CUDA(cub::DeviceSegmentedSort::SortPairs(L.cub_tmp, cbs, mst_b, kout, mst_w, vout, (int)ne, (int)nseg,
                                                     seg_b, seg_e, st));
      }
      LAUNCH(k_copy_segments, (int)std::min<uint32_t>(nseg, 1u << 20), kThreads, st, seg_b, seg_e, nseg, kout, vout,
             mst_b, mst_w);
    }
    KDB_CUDA(cudaMemsetAsync(L.buckets, 0, 256 * sizeof(unsigned long long), st));
    LAUNCH(k_wbuckets, grid_for(ne), kThreads, st, ne, mst_w, L.buckets);
    KDB_CUDA(cudaGetLastError());
  } else {
    KDB_CUDA(cudaMemsetAsync(L.buckets, 0, 256 * sizeof(unsigned long long), st));
  }
  // the forest's total weight: integer bucket counts, so a SUM over ranks is exact
  if (dist_out)
    KDB_TRY(nccl_check(g_nccl.AllReduce(L.buckets, L.buckets, 256, ncclUint64, ncclSum, comm->nccl, st),
                       "ncclAllReduce(weight buckets)"));
  KDB_CUDA(cudaMemcpyAsync(bk, L.buckets, sizeof(bk), cudaMemcpyDeviceToHost, st));
  KDB_CUDA(cudaEventRecord(m.ev[1], st));
  KDB_CUDA(cudaStreamSynchronize(st));
  const double t_fin = elapsed(m.ev[0], m.ev[1]);
  if (g_prof.on) g_prof.drain();
  KDB_TRY(guards_check((const char*)workspace, L.guards, st, "kdb_mst"));
  *mst_count = ne;
  *mst_weight = exact_bucket_sum(bk);
  if (m.ell_next.valid) ell_put(m.ell_next);
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
  // local-first contraction (multi-rank exact mode): per-virtual-rank local
  // phase (max / sum over ranks), transition, global phase, and what the
  // global phase received
  g_stats[19] = m.lf ? 1.0 : 0.0;
  g_stats[20] = m.t_local_max;
  g_stats[21] = m.t_local_sum;
  g_stats[22] = m.t_transition;
  g_stats[23] = m.t_global;
  g_stats[24] = (double)m.C_global;
  g_stats[25] = (double)m.parked_rows;
  g_stats[26] = m.payload_transition;
  g_stats[27] = m.local_rounds;
  g_stats[28] = m.t_global_scan;
  g_stats[29] = m.reused;
  g_stats[30] = m.t_heavy_rank;
  g_stats[31] = m.t_heavy_simred;
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
  // the cut entries live in the survivor buffers, whose counts go to CUB as int
  if (g && g->n_rows * (int64_t)edge_cols_of(g) >= (int64_t)INT32_MAX)
    return set_err(KDB_EINVAL, "kdb_mst_inexact: n_rows * edge_cols must stay below 2^31 - 1");
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
size_t nmi_carve(NmiWs& w, char* base, bool dry, int64_t n, std::vector<size_t>* guards = nullptr) {
  Carver cv{base, 0, 0, dry};
  cv.guards = guards;
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
  ell_take(workspace);  // a light ELL kept in this workspace does not survive this call
  NmiWs w;
  std::vector<size_t> guards;
  const size_t need = nmi_carve(w, (char*)workspace, false, n, &guards);
  if (n > 0 && ws_bytes < need) return set_err(KDB_ENOMEM, "workspace %zu < required %zu bytes", ws_bytes, need);
  *nmi = 1.0;
  *clusters_a = *clusters_b = 0;
  if (n == 0) return KDB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  KDB_TRY(guards_fill((char*)workspace, guards, st));
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
  KDB_TRY(guards_check((const char*)workspace, guards, st, "kdb_nmi"));
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
