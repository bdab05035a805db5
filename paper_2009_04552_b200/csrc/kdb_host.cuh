// kdb_host.cuh -- host side: workspace layout, the rows / filter / heavy phases and the round loop
// Part of kdb.cu's single translation unit: included inside its anonymous
// namespace, after kdb.cu's helpers; not a standalone header.
#pragma once

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
// (n_rows / 2: an eps near the median of D[:, M-1] leaves half the points
// non-core, the light graph fragments and C4 keeps 27.6M survivors -- above
// n_rows / 4 that re-ran the whole rows phase at eps, 40 ms against a few ms of
// heavy rounds; 48 B per row of workspace)
inline int64_t survivor_cap(int64_t n_rows, int64_t k) {
  return std::max<int64_t>(n_rows / 2, std::min<int64_t>(n_rows * k / 4, (int64_t)1 << 24)) + 65536;
}

// Workspace carving.  The debug build (-DKDB_GUARDS=1, lib/libkdb_dbg.so)
// puts a 256-B guard band after every array; kdb_mst / kdb_nmi fill the bands
// with a pattern before their first launch and verify them after the last
// (KDB_EINTERNAL on an overrun) -- the memcheck this pool's GPUs cannot run.
struct Carver {
  char* base;
  size_t off = 0, cap;
  bool dry;
  std::vector<size_t>* guards = nullptr;
  template <typename T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = dry ? nullptr : reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    if (kGuardBytes) {
      off = (off + 255) & ~size_t(255);
      if (guards) guards->push_back(off);
      off += kGuardBytes;
    }
    return p;
  }
};

kdb_status guards_fill(char* base, const std::vector<size_t>& g, cudaStream_t st) {
  for (size_t o : g) KDB_CUDA(cudaMemsetAsync(base + o, kGuardByte, kGuardBytes, st));
  if (!g.empty()) {
    const unsigned int z = 0;
    KDB_CUDA(cudaMemcpyToSymbolAsync(g_dbg_viol, &z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
  }
  return KDB_OK;
}

kdb_status guards_check(const char* base, const std::vector<size_t>& g, cudaStream_t st, const char* what) {
  if (g.empty()) return KDB_OK;
  std::vector<unsigned char> h(kGuardBytes);
  for (size_t i = 0; i < g.size(); ++i) {
    KDB_CUDA(cudaMemcpyAsync(h.data(), base + g[i], kGuardBytes, cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    for (unsigned char c : h)
      if (c != kGuardByte) return set_err(KDB_EINTERNAL, "%s: workspace guard band %zu overwritten", what, i);
  }
  unsigned int viol = 0;
  KDB_CUDA(cudaMemcpyFromSymbolAsync(&viol, g_dbg_viol, sizeof(viol), 0, cudaMemcpyDeviceToHost, st));
  KDB_CUDA(cudaStreamSynchronize(st));
  if (viol) return set_err(KDB_EINTERNAL, "%s: device bounds check failed (mask 0x%x)", what, viol);
  return KDB_OK;
}

struct RankState {
  int64_t row_begin = 0, n_rows = 0;
  const int32_t* nbr = nullptr;
  const float* dist = nullptr;
  Rec* act[2] = {nullptr, nullptr};  // active rows (v, head), ping-pong
  uint32_t n_act = 0;                 // live rows in act[cur]
  uint32_t n_deep = 0;                // rows whose ELL entries are all light (k_light_ell)
  uint32_t n_local = 0;               // rows whose nearest neighbour's id is near their own (k_light_ell)
  bool compact = false;               // rows phase reads the light ELL (else the graph rows)
  int4* LE = nullptr;                 // light ELL: kW/4 planes [kW/4][n_rows] of 32-B chunks ((J, w bits) x 4)
  uint32_t* kthL = nullptr;           // per row: certificate bound kth' of the ELL's threshold (kept for reuse)
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
  // local-first phase (multi-rank exact mode): the phase's own round counters
  // and the rows parked for the global phase (heads kept)
  RoundCounters* lctr = nullptr;
  Rec* park = nullptr;
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
  uint8_t *frz, *frz2;  // local-first phase: frozen components (ping-pong through the contraction)
  int32_t* hcomp;   // heavy phase: light component -> heavy component
  int32_t* dom;     // filter fast path: dominant component per id block
  int2* brun;       // filter fast path: id range of the run of equal-dom blocks around each block
  uint32_t* bloom;  // filter fast path: Bloom filter of the exceptions
  unsigned long long* fcount;  // [0] exceptions, [1] slow-path entries
  float* tau_sample;
  RoundCounters* ctr;
  void* cub_tmp;
  size_t cub_bytes;
  std::vector<RankState> ranks;
  std::vector<size_t> guards;  // debug build: guard band offsets
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
  size_t h3 = 0, g3 = 0;
  cub::DeviceSegmentedSort::SortPairs(nullptr, g3, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                      (const float*)nullptr, (float*)nullptr, (int)std::max<int64_t>(N + 1, 1),
                                      (int)std::max<int64_t>(N / (kRunMax + 1) + 1, 1), (const int32_t*)nullptr,
                                      (const int32_t*)nullptr);
  f = std::max(f, g3);
  cub::DeviceSelect::Flagged(nullptr, h3, (const HEdge*)nullptr, (const uint8_t*)nullptr, (HEdge*)nullptr,
                             (uint32_t*)nullptr, (int)std::min<int64_t>(survivor_cap(N, 65535) + 1, INT32_MAX));
  f = std::max(f, h3);
  return std::max(std::max(a, f), std::max(b, c)) + 256;
}

// carve the workspace; returns bytes needed
size_t carve(Layout& L, char* base, bool dry, int64_t N, int nr, const int64_t* rb, const int64_t* rn,
             bool general, int32_t k, int64_t hs_cap_override = -1, bool local_first = false) {
  Carver cv{base, 0, 0, dry};
  L.guards.clear();
  cv.guards = &L.guards;
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
  L.frz = local_first ? cv.take<uint8_t>(N + 1) : nullptr;
  L.frz2 = local_first ? cv.take<uint8_t>(N + 1) : nullptr;
  L.hcomp = cv.take<int32_t>(N + 1);
  L.dom = cv.take<int32_t>(kDomMax);
  L.brun = cv.take<int2>(kDomMax);
  L.bloom = cv.take<uint32_t>(kBloomBits / 32);
  L.fcount = cv.take<unsigned long long>(2);
  L.tau_sample = cv.take<float>(kTauSamples);
  L.ctr = cv.take<RoundCounters>(2);  // [1]: rank 0's counters (one snapshot copy for both)
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
    R.kthL = general ? nullptr : cv.take<uint32_t>(n);
    R.off_cap_rows = n;
    R.offers = cv.take<Offer>(general ? n + N : n);
    R.ctr = r == 0 ? L.ctr + 1 : cv.take<RoundCounters>(1);
    if (local_first) {  // local-first phase (exact mode, > 1 rank)
      R.lctr = cv.take<RoundCounters>(1);
      R.park = cv.take<Rec>(n);
    }
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
                                           (int64_t)INT32_MAX - 1);  // CUB item counts are int
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
  if (g->flags & ~(KDB_GRAPH_EXACT | KDB_GRAPH_REUSE)) return set_err(KDB_EINVAL, "unknown graph flags");
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

// Collectives run with a real NCCL communicator of > 1 rank -- or, with the
// option KDB_NCCL_FORCE = 1 (tests, bench --nccl1), on a 1-rank NCCL communicator too, so one GPU runs
// the multi-rank host logic (exact per-round counts, agreed branches) through
// real NCCL calls.
bool multi_rank(const kdb_comm* comm) {
  if (!comm || comm->kind != 1) return false;
  if (comm->nranks > 1) return true;
  return opt_int("KDB_NCCL_FORCE", 0) != 0;
}


// Local-first contraction runs when more than one rank shares
// the graph (a real NCCL communicator, the sim communicator with P >= 2, or the
// forced 1-rank NCCL test mode) and the caller promises an exact graph (the
// certificate is what lets a rank decide from its own rows); KDB_LOCAL=0 turns
// it off (the replicated-rounds path of round 1).
bool local_first_on(const kdb_graph* g, const kdb_comm* comm) {
  if (!(g->flags & KDB_GRAPH_EXACT) || opt_int("KDB_LOCAL", 1) == 0) return false;
  if (opt_int("KDB_COMPACT", 1) == 0 || opt_int("KDB_FUSE1", 1) == 0 || opt_int("KDB_CAS", 1) == 0 ||
      opt_int("KDB_PACK1", 1) == 0)
    return false;  // the phase runs on the one-rank machinery (ELL, fused round 1, CAS offers)
  return multi_rank(comm) || (comm && comm->kind == 2 && comm->nranks >= 2);
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


bool nr_ranks_is_one(const Layout& L) { return L.ranks.size() == 1; }

// What a kept light ELL was built from.  The ELL (first kW entries of every
// row) and the per-row certificate bounds depend on the graph and on the
// rows-phase threshold eps_run only -- for the light phase that is tau, the
// median of a fixed column, not eps -- so an eps sweep over one graph can skip
// the ELL pass after its first call.  Host-side table keyed by the workspace.
struct EllKey {
  bool valid = false;
  const void* ws = nullptr;
  const int32_t* nbr = nullptr;
  const float* dist = nullptr;
  int64_t n_total = 0, row_begin = 0, n_rows = 0;
  int32_t k_max = 0, k = 0;
  uint32_t eps_run_bits = 0, n_deep = 0, n_local = 0;
  bool same_graph(const EllKey& o) const {
    return ws == o.ws && nbr == o.nbr && dist == o.dist && n_total == o.n_total && row_begin == o.row_begin &&
           n_rows == o.n_rows && k_max == o.k_max && k == o.k;
  }
};
std::mutex g_ell_mu;
std::vector<EllKey> g_ell;  // at most a few workspaces in flight
EllKey ell_take(const void* ws) {  // remove and return the entry of this workspace
  std::lock_guard<std::mutex> lk(g_ell_mu);
  EllKey out;
  for (size_t i = 0; i < g_ell.size(); ++i)
    if (g_ell[i].ws == ws) {
      out = g_ell[i];
      g_ell.erase(g_ell.begin() + i);
      break;
    }
  return out;
}
void ell_put(const EllKey& e) {
  std::lock_guard<std::mutex> lk(g_ell_mu);
  if (g_ell.size() >= 64) g_ell.erase(g_ell.begin());
  g_ell.push_back(e);
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
  // local-first contraction: lf = run it (multi-rank exact
  // mode); local = this Mst is one rank's local phase (view lv, C0 local
  // components, MSF slots ecap); cont = the global phase continuing from the
  // parked rows
  bool lf = false, local = false, cont = false;
  LocalView lv;
  int64_t C0 = 0, ecap = -1;
  uint64_t n_park = 0, msf_local = 0;
  double t_local_max = 0, t_local_sum = 0, t_transition = 0, t_global = 0;
  int local_rounds = 0;
  // light ELL kept across calls on one workspace (KDB_GRAPH_REUSE, eps sweeps)
  bool reuse_req = false;
  const void* ws = nullptr;   // the caller's workspace (key of the kept-ELL table)
  EllKey ell_prev, ell_next;  // what the previous call left / what this call leaves (valid flags inside)
  int reused = 0;             // rows phases that reused the kept ELL
  double t_global_scan = 0;  // global phase: per-rank offers and ties (all ranks, in sequence under sim)
  double t_heavy_rank = 0;   // heavy phase: per-rank survivor offers, compaction and ties (all ranks)
  double t_heavy_simred = 0; // heavy phase: the sim communicator's min-reductions (an all-reduce on GPUs)
  int64_t C_global = -1;      // components entering the global phase
  uint64_t parked_rows = 0;   // rows entering the global phase (all ranks)
  double payload_transition = 0;  // bytes per rank of the all-gathers between the phases
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

kdb_status local_first(Mst& m, float eps_run);

// Records per block chunk of the ordered row kernels (and components per hook
// chunk): kChunk = 1024 for long lists; short lists use smaller chunks so a
// thread scans one record instead of four in sequence (small inputs are
// latency-bound: C1's light rounds took ~40 us each with 1,024-record chunks)
inline int row_chunk(uint64_t n) { return n >= (1ull << 21) ? kChunk : n >= (1ull << 19) ? 512 : 256; }

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
  const bool use_compact = opt_int("KDB_COMPACT", 1) != 0;
  const int gw = opt_int("KDB_GW", 4);  // component-gather width of the later light rounds (scan_ell)
  const bool lean = opt_int("KDB_LEAN", 0) != 0;  // chunk scan on bit masks (scan_ell_lean): measured slower, off
  const bool sparse_ids = opt_int("KDB_SPARSE", 1) != 0;  // keep root ids once few components remain
  const int skip1 = opt_int("KDB_SKIP1", 1);  // round-2 heads skip the entry round 1 hooked along
  // bit 0: evict-last L2 policy on the light rounds' component gathers; bit 1:
  // those gathers through L1 (KDB_L1GAT)
  // (KDB_L1GAT; default: when most rows' nearest neighbour has a nearby id, k_light_ell counts them)
  int l2hint = (opt_int("KDB_L2HINT", 1) ? 1 : 0) | (opt_int("KDB_L1GAT", 0) > 0 ? 2 : 0);
  const int l1gat_env = opt_int("KDB_L1GAT", -1);
  // local-first phase of one rank (m.local): LOCAL component ids, the rank's
  // per-component slices, no exchange; the global phase (m.cont) continues the
  // rounds from the rows the local phases parked
  LocalView lv = m.local ? m.lv : LocalView{};
  uint8_t* frz = m.local ? L.frz : nullptr;
  const int64_t ecap = m.ecap >= 0 ? m.ecap : N;
  int64_t C = 0;
  bool fuse1 = false, packed1 = false, packed1r = false, tile = false;
  size_t cb = L.cub_bytes;
  int32_t* gmap = nullptr;   // two-level ids in the global phase (LocalView::gmap)
  int64_t CG0 = 0;
  if (m.cont) {
    C = m.C;  // global components after the local-first phases (state set by local_first)
    if (opt_int("KDB_GMAP", 1) != 0 && C > 0) {
      gmap = L.hcomp;  // free until the heavy phase
      CG0 = C;
      LAUNCH(k_iota, grid_for(C), kThreads, st, gmap, C);
      lv.gmap = gmap;
    }
  } else {
  KDB_CUDA(cudaMemsetAsync(L.ctr, 0, sizeof(RoundCounters), st));
  if (!m.local) {
    // ---- a2: dense component ids -------------------------------------------------
    const int64_t nwords = (N + 31) / 32;
    uint32_t* popc = reinterpret_cast<uint32_t*>(L.flag);  // scratch, nwords + 1 <= N + 1
    KDB_CUDA(cudaMemsetAsync(popc + nwords, 0, sizeof(uint32_t), st));
    LAUNCH(k_popc_words, grid_for(nwords), kThreads, st, core_bits, nwords, popc);
    KDB_CUDA(cudaGetLastError());
    { LaunchScope ls_("cub::DeviceScan", st, false); KDB_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb, popc, L.woff, (int)(nwords + 1), st)); }
    uint32_t C32 = 0;  // woff[nwords] = number of core points
    KDB_CUDA(cudaMemcpyAsync(&C32, L.woff + nwords, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    C = C32;
    L.all_core = (C == N) ? 1 : 0;  // then the dense id of a vertex is the vertex itself
    LAUNCH(k_init_comp, grid_for(N), kThreads, st, core_bits, L.woff, N, comp, L.cmin);
    if (m.lf) return local_first(m, eps_run);
  } else {
    // local ids: dense over this rank's core rows (the caller shifted comp)
    C = m.C0;
    L.all_core = (C == L.ranks[0].n_rows) ? 1 : 0;  // then a row's local id is v - lo
    KDB_CUDA(cudaMemsetAsync(frz, 0, (size_t)std::max<int64_t>(C, 1), st));
  }
  // eps sweep on an unchanged graph: reuse the ELL the previous call kept
  const bool one_rank = L.ranks.size() == 1 && !multi_rank(comm) && !m.local;
  uint32_t eb = 0;
  memcpy(&eb, &eps_run, 4);
  EllKey want;
  if (one_rank && !general && use_compact) {
    const RankState& R0 = L.ranks[0];
    want.valid = true;
    want.ws = m.ws;
    want.nbr = R0.nbr;
    want.dist = R0.dist;
    want.n_total = N;
    want.row_begin = R0.row_begin;
    want.n_rows = R0.n_rows;
    want.k_max = ld;
    want.k = k;
    want.eps_run_bits = eb;
  }
  const bool reuse = want.valid && m.reuse_req && m.ell_prev.valid && m.ell_prev.same_graph(want) &&
                     m.ell_prev.eps_run_bits == eb && L.ranks[0].n_rows > 0;
  // exact mode: round 1 (singleton components) is fused into the ELL pass; a
  // single rank also packs (K, B, kmin) per component for the round-1 hook
  // (with a reused ELL round 1 runs over it: k_light_first)
  // tile round (one rank, exact mode, light ELL): round 1 is tile-local
  // Boruvka in shared memory (k_tile_round) instead of the fused singleton round
  tile = want.valid && want.row_begin == 0 && opt_int("KDB_TILE", 0) != 0 && L.ranks[0].n_rows > 0;
  fuse1 = !general && use_compact && opt_int("KDB_FUSE1", 1) != 0 && !reuse && !tile;
  packed1 = fuse1 && L.ranks.size() == 1 && !(multi_rank(comm)) && opt_int("KDB_PACK1", 1) != 0;
  // a reused ELL (eps sweep): round 1 over it (k_light_first) writes the same
  // packed records, and k_reuse_rows the sentinel records of the other components
  packed1r = reuse && L.rec1 && opt_int("KDB_PACK1", 1) != 0;
  // Per-component slots of round 1.  Packed round 1 (one rank, fused ELL pass)
  // writes a whole record and the certificate bound for EVERY component (each
  // is one core row of this rank) and the hook reads tgt only under a finite
  // key: nothing to initialise.
  if (!packed1 && !packed1r) {
    LAUNCH(k_fill_comp_arrays, grid_for(C), kThreads, st, C, L.Kc, L.Bc, general ? nullptr : L.kmin);
    for (size_t r = 1; r < L.ranks.size(); ++r)
      LAUNCH(k_fill_comp_arrays, grid_for(C), kThreads, st, C, L.ranks[r].Kc, L.ranks[r].Bc, nullptr);
    if (!general)  // hook targets of round 1 (written by the round-1 offers)
      for (auto& R : L.ranks) LAUNCH(k_fill_i32, grid_for(C), kThreads, st, R.tgt, C, INT32_MAX);
  }
  KDB_CUDA(cudaGetLastError());
  for (auto& R : L.ranks) {
    KDB_CUDA(cudaMemsetAsync(R.ctr, 0, sizeof(RoundCounters), st));
    R.compact = false;
    if (reuse) {
      R.compact = true;
      LAUNCH(k_reuse_rows, grid_for(R.n_rows), kThreads, st, R.LE, R.kthL, R.n_rows, R.row_begin, eps_run, comp,
             L.kmin, R.act[0], &R.ctr->na[0], packed1r ? L.rec1 : (int4*)nullptr);
      ++m.reused;
    } else if (R.n_rows > 0 && use_compact) {
      R.compact = true;
      // 32-byte sector loads need 32-B aligned arrays, ld % 8 in {0, 4} and rows
      // long enough for the third sector (ld >= 20)
      const bool a32 = vec && ld >= 20 && !(((uintptr_t)R.nbr | (uintptr_t)R.dist) & 31u);
#define KDB_ELL_LAUNCH(V, A)                                                                                    \
  LAUNCH((k_light_ell<V, A>), grid_for(R.n_rows), kThreads, st, R.nbr, R.dist, R.n_rows, ld, k, eps_run, R.row_begin, \
         comp, general ? nullptr : L.kmin, R.LE, R.act[0], &R.ctr->na[0], &R.ctr->grab, fuse1 ? 1 : 0,         \
         L.all_core, N, R.Kc, R.Bc, R.tgt, packed1 ? L.rec1 : nullptr, &R.ctr->n_deep, lv, skip1,               \
         row_chunk((uint64_t)R.n_rows), want.valid ? R.kthL : (uint32_t*)nullptr)
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
  if (!general && !m.local) m.payload_rows += 4.0 * C;
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
    R.n_deep = reuse ? m.ell_prev.n_deep : hc.n_deep;
    R.n_local = reuse ? m.ell_prev.n_local : hc.n_local;
    R.n_in_act = hc.ni[0];
  }
  if (want.valid) {  // what this call's ELL was built from (kept if the call succeeds)
    m.ell_next = want;
    m.ell_next.n_deep = L.ranks[0].n_deep;
    m.ell_next.n_local = L.ranks[0].n_local;
  }
  KDB_CUDA(cudaEventRecord(ev[2], st));
  KDB_CUDA(cudaEventSynchronize(ev[2]));
  m.t_init += elapsed(ev[0], ev[1]);
  m.t_inlist += elapsed(ev[1], ev[2]);
  }  // !m.cont

  if (l1gat_env < 0) {  // auto: spatially ordered ids (e.g. the inertial partition)
    uint64_t loc = 0, rows = 0;
    for (auto& R : L.ranks) {
      loc += R.n_local;
      rows += (uint64_t)std::max<int64_t>(R.n_rows, 0);
    }
    if (rows > 0 && 2 * loc > rows) l2hint |= 2;
  }
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
  // one rank, exact mode, light ELL: rounds >= 2 offer by a 128-bit CAS-minimum
  // of (key, b) (no offer list, no tie pass); KB reuses the round-1 records
  // (rec1: 16 B per component, free once round 1 has hooked)
  const bool cas = !general && nr_ranks_is_one(L) && !multi_rank(comm) && any_compact && L.rec1 &&
                   opt_int("KDB_CAS", 1) != 0;
  ulonglong2* KB = cas ? reinterpret_cast<ulonglong2*>(L.rec1) : nullptr;
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
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> gscan;  // global phase: per-rank work spans
  const uint32_t* kmin_cert = general ? nullptr : L.kmin;
  auto slot_of = [&](int rr) { return slots + (size_t)(rr % kSlots) * (1 + nr); };

  // contraction a6 on the device counts; C_bound >= the true count
  auto contract = [&](int64_t C_bound) -> kdb_status {
    const int64_t* Cd = (const int64_t*)&L.ctr->Cs[par];
    int64_t* Cn = (int64_t*)&L.ctr->Cs[par ^ 1];
    // sparse ids once few components remain: a component keeps its root's id
    // (no dense renumbering; the id range stays C_bound), so the relabel only
    // rewrites the vertices of merged components
    const bool sparse = sparse_ids && C_bound <= N / 64;
    LAUNCH(k_jump, grid_for(C_bound), kThreads, st, C_bound, L.parent, L.rootof, L.ctr, Cd,
           sparse ? (int32_t*)nullptr : L.flag);
    if (!sparse) {
      size_t cb2 = L.cub_bytes;
      { LaunchScope ls_("cub::DeviceScan", st, false); KDB_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb2, L.flag, L.newid, (int)std::max<int64_t>(C_bound, 1), st)); }
    }
    // new count + next round's slots (cmin2 / kmin2 before k_merge; the offer
    // slots are free: the hook has read them)
    LAUNCH(k_round_fill, grid_for(C_bound), kThreads, st, C_bound, Cd, sparse ? (const int32_t*)nullptr : L.newid,
           (const int32_t*)L.flag, Cn, L.cmin2, general ? (uint32_t*)nullptr : L.kmin2, L.Kc, L.Bc, KB,
           frz ? L.frz2 : (uint8_t*)nullptr);
    // map[c] = new dense id of c's tree (reuses `parent`, no longer needed)
    LAUNCH(k_merge, grid_for(C_bound), kThreads, st, C_bound, L.rootof, sparse ? (const int32_t*)nullptr : L.newid,
           L.cmin, general ? nullptr : L.kmin, L.cmin2, L.kmin2, L.parent, Cd, (const uint8_t*)frz,
           frz ? L.frz2 : nullptr);
    if (m.local)  // only this rank's rows carry (local) ids
      LAUNCH(k_relabel, grid_for((lv.hi - lv.lo) / 8 + 1), kThreads, st, lv.hi - lv.lo, comp + lv.lo, L.parent,
             (const int32_t*)nullptr);
    else if (gmap)  // global phase: the map of transition ids, not the N vertices
      LAUNCH(k_relabel, grid_for(CG0 / 8 + 1), kThreads, st, CG0, gmap, L.parent, (const int32_t*)nullptr);
    else
      LAUNCH(k_relabel, grid_for(N / 8 + 1), kThreads, st, N, comp, L.parent, (const int32_t*)nullptr);
    // ranks >= 1 of a sim communicator: their partial offer slots (on GPUs each
    // rank refills only its own -- k_round_fill above): timed as per-rank work
    cudaEvent_t fa = nullptr, fb = nullptr;
    if (m.cont && nr > 1) {
      KDB_CUDA(cudaEventCreate(&fa));
      KDB_CUDA(cudaEventCreate(&fb));
      ev_rnd.push_back(fa);
      ev_rnd.push_back(fb);
      KDB_CUDA(cudaEventRecord(fa, st));
    }
    for (size_t r = 1; r < nr; ++r)
      LAUNCH(k_fill_comp_arrays, grid_for(C_bound), kThreads, st, C_bound, L.ranks[r].Kc, L.ranks[r].Bc, nullptr,
             (const int64_t*)Cn);
    if (fa) {
      KDB_CUDA(cudaEventRecord(fb, st));
      gscan.push_back({fa, fb});
    }
    KDB_CUDA(cudaGetLastError());
    std::swap(L.cmin, L.cmin2);
    std::swap(L.kmin, L.kmin2);
    if (frz) {
      std::swap(L.frz, L.frz2);
      frz = L.frz;
    }
    kmin_cert = general ? nullptr : L.kmin;
    par ^= 1;
    return KDB_OK;
  };
  // snapshot of the counters after the current round into a pinned slot
  auto snapshot = [&](int rr) -> kdb_status {
    RoundCounters* sl = slot_of(rr);
    // the global counters and rank 0's are adjacent in the workspace (carve):
    // one copy for both in the one-rank case
    const size_t r0 = L.ranks[0].ctr == L.ctr + 1 ? 1 : 0;
    KDB_CUDA(cudaMemcpyAsync(sl, L.ctr, (1 + r0) * sizeof(RoundCounters), cudaMemcpyDeviceToHost, st));
    for (size_t r = r0; r < nr; ++r)
      KDB_CUDA(cudaMemcpyAsync(sl + 1 + r, L.ranks[r].ctr, sizeof(RoundCounters), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaEventRecord(ev_slot[rr % kSlots], st));
    return KDB_OK;
  };

  int last_checked = 0;
  bool finished = false;
  while (!finished) {
    ++rounds;
    const bool direct = rounds == 1 && !general && !m.cont;
    const int64_t* Cd = (const int64_t*)&L.ctr->Cs[par];
    if (ev_rnd.empty()) {  // the phase's start (rounds are pipelined: timed as one span)
      cudaEvent_t e0;
      KDB_CUDA(cudaEventCreate(&e0));
      ev_rnd.push_back(e0);
      KDB_CUDA(cudaEventRecord(e0, st));
    }
    const bool tile_round = tile && rounds == 1;
    if (tile_round) {  // round 1: tile-local Boruvka (kdb_tile.cuh); then contract as after any round
      RankState& R = L.ranks[0];
      KDB_CUDA(cudaMemsetAsync(&R.ctr->na[cur ^ 1], 0, sizeof(uint32_t), st));
      KDB_CUDA(cudaMemsetAsync(&R.ctr->grab, 0, sizeof(uint32_t), st));
      KDB_CUDA(cudaMemsetAsync(&L.ctr->hooks, 0, 4 * sizeof(uint32_t), st));
#define KDB_TILE_LAUNCH(T)                                                                                     \
  LAUNCH_DYN(k_tile_round<T>, (int)std::min<int64_t>((R.n_rows + (T) - 1) / (T), 1 << 30), (T),                 \
             sizeof(TileSmem<T>), st, R.LE, R.n_rows, k, eps_run, N, comp, core_bits, L.kmin, L.parent, L.e_key, \
             L.e_w, ecap, R.act[cur ^ 1], &R.ctr->na[cur ^ 1], &R.ctr->grab, L.ctr, &L.ctr->entries,      \
             std::max(1, std::min(opt_int("KDB_TILE_MAXR", kTileMaxRounds), kTileMaxRounds)))
      if (opt_int("KDB_TILE_ROWS", 1024) == 512) KDB_TILE_LAUNCH(512);
      else KDB_TILE_LAUNCH(1024);
#undef KDB_TILE_LAUNCH
      KDB_CUDA(cudaGetLastError());
    } else {
    // offers read the current key before their atomicMin once many rows offer
    // to each component (same-address atomics serialise; early rounds have
    // about one row per component and only pay the extra read)
    int precheck = 0;
    {
      uint64_t live = 0;
      for (size_t r = 0; r < nr; ++r) live += na_ub[r];
      const int pc = opt_int("KDB_PRECHECK", -1);
      precheck = pc >= 0 ? pc : (live > 8 * (uint64_t)std::max<int64_t>(C_ub, 1) ? 1 : 0);
    }
    // global phase of the local-first scheme: time the per-rank work (offers,
    // ties: divides by the rank count on real GPUs) apart from the rest
    cudaEvent_t gsA = nullptr, gsB = nullptr, gsC = nullptr, gsD = nullptr;
    if (m.cont) {
      for (cudaEvent_t* e : {&gsA, &gsB, &gsC, &gsD}) {
        KDB_CUDA(cudaEventCreate(e));
        ev_rnd.push_back(*e);
      }
      KDB_CUDA(cudaEventRecord(gsA, st));
    }
    // a3: offers (rows, then in-lists), per rank, into that rank's Kc partial
    bool hooks_zeroed = false;
    for (size_t r = 0; r < nr; ++r) {
      RankState& R = L.ranks[r];
      if (direct && fused && R.compact) continue;  // done by the ELL pass
      // this round's counters (and, with rank 0, the hook counters: nothing
      // writes them before the hook) in one launch instead of five memsets
      LAUNCH(k_round_reset, 1, 32, st, R.ctr, cur, r == 0 ? L.ctr : (RoundCounters*)nullptr);
      hooks_zeroed |= r == 0;
      const uint32_t* nin = &R.ctr->na[cur];
      uint32_t* nout = &R.ctr->na[cur ^ 1];
      if (na_ub[r] && R.compact) {
        if (direct)
          LAUNCH(k_light_first, grid_for(na_ub[r]), kThreads, st, R.LE, R.n_rows, R.nbr, R.dist, ld, k, eps_run, R.row_begin, N,
                 comp, L.all_core, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, R.Kc, R.Bc, R.tgt,
                 &L.ctr->entries, nin, row_chunk(na_ub[r]), packed1r ? L.rec1 : (int4*)nullptr, R.kthL, skip1);
        else
        {
#define KDB_LR_LAUNCH(...)                                                                                       \
  LAUNCH((k_light_round<__VA_ARGS__>), grid_for(na_ub[r]), kThreads, st, R.LE, R.n_rows, R.nbr, R.dist, ld, k, eps_run,       \
         R.row_begin, N, comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, R.offers,                 \
         (unsigned long long*)R.Kc, &L.ctr->entries, nin, precheck, KB, lv, (const uint8_t*)frz, R.park,         \
         m.local ? &L.ctr->n_park : nullptr, l2hint, row_chunk(na_ub[r]))
          // pipelined chunk loads pay when many rows scan past their first chunk
          // (C3: its inner shell is all light); they cost occupancy otherwise
          const int pk = opt_int("KDB_PIPE", -1);
          // KDB_PIPE_R0..KDB_PIPE_R1 (experiment): pipelined loads in those rounds only
          const int pr0 = opt_int("KDB_PIPE_R0", 0), pr1 = opt_int("KDB_PIPE_R1", -1);
          const bool pipe = pk >= 0 ? pk != 0
                                    : (rounds >= pr0 && rounds <= pr1) ||
                                          (uint64_t)R.n_deep * 100 > (uint64_t)R.n_rows * 15;
          // the gather's view fixed at compile time when it is the plain one
          // (no rank window, no global map): KDB_GM = 0 keeps the runtime view
          const int gm = (!lv.bits && !lv.gmap && opt_int("KDB_GM", 1) != 0)
                             ? ((l2hint & 2) ? (int)kGmL1 : (l2hint & 1) ? (int)kGmHint : (int)kGmRuntime)
                             : (int)kGmRuntime;
          const bool fast_scan = opt_int("KDB_FASTSCAN", 0) != 0;  // scan_ell_fast: measured slower (10.65 vs 10.16 ms), off
          // lane refill (k_light_refill): the one-view CAS case without pipelined
          // loads; parity-green but measured 2.7x slower (C4: 27.6 vs 10.2 ms), off
          const bool refill = cas && !pipe && !lean && gm != kGmRuntime && !frz && opt_int("KDB_REFILL", 0) != 0;
          // quad per row (k_light_quad): the same one-view CAS case; parity-green but
          // measured 3.5x slower (C4: 35.4 vs 10.2 ms of light rounds, same box), off
          const bool quad = !refill && cas && !pipe && !lean && gm != kGmRuntime && !frz && opt_int("KDB_QUAD", 0) != 0;
          // level-synchronous chunk scan (k_light_lvl): the same one-view CAS case
          const bool lvl = !refill && cas && !pipe && !lean && gm != kGmRuntime && !frz && opt_int("KDB_LVL", 0) != 0;
          if (lvl && opt_int("KDB_LVL", 0) == 3) {  // pooled variant with the branch-free chunk scan
            if (gm == kGmL1)
              LAUNCH((k_light_pool<kGmL1, true>), grid_for(na_ub[r]), kThreads, st, R.LE, R.n_rows, R.nbr, R.dist, ld, k,
                     eps_run, R.row_begin, N, comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, KB,
                     &L.ctr->entries, nin, l2hint, row_chunk(na_ub[r]));
            else
              LAUNCH((k_light_pool<kGmHint, true>), grid_for(na_ub[r]), kThreads, st, R.LE, R.n_rows, R.nbr, R.dist, ld, k,
                     eps_run, R.row_begin, N, comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, KB,
                     &L.ctr->entries, nin, l2hint, row_chunk(na_ub[r]));
          } else if (lvl && opt_int("KDB_LVL", 0) == 2) {  // pooled variant (k_light_pool)
            if (gm == kGmL1)
              LAUNCH(k_light_pool<kGmL1>, grid_for(na_ub[r]), kThreads, st, R.LE, R.n_rows, R.nbr, R.dist, ld, k,
                     eps_run, R.row_begin, N, comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, KB,
                     &L.ctr->entries, nin, l2hint, row_chunk(na_ub[r]));
            else
              LAUNCH(k_light_pool<kGmHint>, grid_for(na_ub[r]), kThreads, st, R.LE, R.n_rows, R.nbr, R.dist, ld, k,
                     eps_run, R.row_begin, N, comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, KB,
                     &L.ctr->entries, nin, l2hint, row_chunk(na_ub[r]));
          } else if (lvl) {
            if (gm == kGmL1)
              LAUNCH(k_light_lvl<kGmL1>, grid_for(na_ub[r]), kThreads, st, R.LE, R.n_rows, R.nbr, R.dist, ld, k,
                     eps_run, R.row_begin, N, comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, KB,
                     &L.ctr->entries, nin, l2hint, row_chunk(na_ub[r]));
            else
              LAUNCH(k_light_lvl<kGmHint>, grid_for(na_ub[r]), kThreads, st, R.LE, R.n_rows, R.nbr, R.dist, ld, k,
                     eps_run, R.row_begin, N, comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, KB,
                     &L.ctr->entries, nin, l2hint, row_chunk(na_ub[r]));
          } else if (quad) {
            if (gm == kGmL1)
              LAUNCH(k_light_quad<kGmL1>, grid_for(na_ub[r]), kThreads, st, R.LE, R.n_rows, R.nbr, R.dist, ld, k,
                     eps_run, R.row_begin, N, comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, KB,
                     &L.ctr->entries, nin, l2hint, row_chunk(na_ub[r]));
            else
              LAUNCH(k_light_quad<kGmHint>, grid_for(na_ub[r]), kThreads, st, R.LE, R.n_rows, R.nbr, R.dist, ld, k,
                     eps_run, R.row_begin, N, comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, KB,
                     &L.ctr->entries, nin, l2hint, row_chunk(na_ub[r]));
          } else if (refill) {
#define KDB_RF_LAUNCH(G)                                                                                          \
  LAUNCH(k_light_refill<G>, grid_for(na_ub[r]), kThreads, st, R.LE, R.n_rows, R.nbr, R.dist, ld, k, eps_run,         \
         R.row_begin, N, comp, R.act[cur], na_ub[r], R.act[cur ^ 1], nout, &R.ctr->grab, KB, &L.ctr->entries, nin, \
         l2hint)
            if (gm == kGmL1) KDB_RF_LAUNCH(kGmL1);
            else KDB_RF_LAUNCH(kGmHint);
#undef KDB_RF_LAUNCH
          } else if (cas) {
            if (pipe) {
              if (gm == kGmL1) KDB_LR_LAUNCH(4, true, true, false, kGmL1);
              else if (gm == kGmHint) KDB_LR_LAUNCH(4, true, true, false, kGmHint);
              else KDB_LR_LAUNCH(4, true, true);
            } else if (lean) KDB_LR_LAUNCH(4, false, true, true);
            else if (gm == kGmL1 && fast_scan) KDB_LR_LAUNCH(4, false, true, false, kGmL1, true);
            else if (gm == kGmHint && fast_scan) KDB_LR_LAUNCH(4, false, true, false, kGmHint, true);
            else if (gm == kGmL1) KDB_LR_LAUNCH(4, false, true, false, kGmL1);
            else if (gm == kGmHint) KDB_LR_LAUNCH(4, false, true, false, kGmHint);
            else KDB_LR_LAUNCH(4, false, true);
          } else if (gw == 1) KDB_LR_LAUNCH(1);
          else if (gw == 2) KDB_LR_LAUNCH(2);
          else if (pipe) KDB_LR_LAUNCH(4, true);
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
    if (m.cont) KDB_CUDA(cudaEventRecord(gsB, st));
    // exchange: sim -> min over virtual ranks; nccl -> allreduce
    for (size_t r = 1; r < nr; ++r)
      LAUNCH(k_min_into_u64, grid_for(C_ub), kThreads, st, L.Kc, L.ranks[r].Kc, C_ub, Cd);
    KDB_TRY(allreduce_min_u64(comm, L.Kc, C_ub, st));
    m.payload_rows += 8.0 * C_ub;
    if (m.cont) KDB_CUDA(cudaEventRecord(gsC, st));
    // a4: ties (the direct round already wrote Bc and the targets)
    if (!direct && !cas) {
      for (size_t r = 0; r < nr; ++r) {
        RankState& R = L.ranks[r];
        if (na_ub[r]) LAUNCH(k_tie, grid_for(na_ub[r]), kThreads, st, R.offers, &R.ctr->na[cur ^ 1], L.Kc, R.Bc);
        if (general && ni_ub[r])
          LAUNCH(k_tie, grid_for(ni_ub[r]), kThreads, st, R.offers + R.off_cap_rows, &R.ctr->n_off, L.Kc, R.Bc);
        KDB_CUDA(cudaGetLastError());
      }
    }
    if (m.cont) {
      KDB_CUDA(cudaEventRecord(gsD, st));
      gscan.push_back({gsA, gsB});
      gscan.push_back({gsC, gsD});
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
    if (!hooks_zeroed) KDB_CUDA(cudaMemsetAsync(&L.ctr->hooks, 0, 4 * sizeof(uint32_t), st));
    if (direct && (packed1 || packed1r))
      LAUNCH(k_hook<true>, grid_for(C_ub), kThreads, st, C_ub, L.Kc, L.Bc, L.tgt, kmin_cert, comp, L.parent, L.e_key,
             L.e_w, ecap, L.ctr, Cd, L.rec1, (const ulonglong2*)nullptr, frz, row_chunk((uint64_t)C_ub));
    else
      LAUNCH(k_hook<false>, grid_for(C_ub), kThreads, st, C_ub, L.Kc, L.Bc, direct ? L.tgt : nullptr, kmin_cert,
             comp, L.parent, L.e_key, L.e_w, ecap, L.ctr, Cd, (const int4*)nullptr,
             (cas && !direct) ? (const ulonglong2*)KB : nullptr, frz, row_chunk((uint64_t)C_ub), lv.gmap);
    KDB_CUDA(cudaGetLastError());
    }  // !tile_round
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
    if (trace_on())
      fprintf(stderr, "[kdb] round %d eps=%.6g C->%lld offered=%u hooks=%u live=%u entries=%llu\n", check,
              (double)eps_run, (long long)g.Cs[(check & 1) ? 1 : 0], g.offered, g.hooks,
              slot_of(check)[1].na[check & 1], (unsigned long long)g.entries);
    if (g.violation == 2u) return set_err(KDB_EINTERNAL, "pointer jumping did not converge (hook cycle)");
    if (g.violation) return set_err(KDB_EINVAL, "graph violates the KDB_GRAPH_EXACT promise (a component's "
                                    "minimum missed an incident edge)");
    if (g.offered == 0) break;  // a8: no component has a leaving edge
    // local-first phase: no hook means every component with a leaving edge is
    // frozen (remote or uncertifiable minimum) -- the rest is the global phase's
    if (m.local && g.hooks == 0) break;
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
      if (gmap) {  // the sweep reads comp[] directly: current ids into comp, the map back to identity
        LAUNCH(k_relabel, grid_for(N / 8 + 1), kThreads, st, N, comp, gmap, (const int32_t*)nullptr);
        LAUNCH(k_iota, grid_for(CG0), kThreads, st, gmap, CG0);
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
  if (gmap)  // the global phase's current ids into comp (the filter and labels read comp)
    LAUNCH(k_relabel, grid_for(N / 8 + 1), kThreads, st, N, comp, gmap, (const int32_t*)nullptr);
  KDB_CUDA(cudaStreamSynchronize(st));
  if (!ev_rnd.empty()) {
    KDB_CUDA(cudaEventRecord(ev[2], st));
    KDB_CUDA(cudaEventSynchronize(ev[2]));
    m.t_min_edges += elapsed(ev_rnd.front(), ev[2]);  // rounds are pipelined: one span
    for (auto& pr : gscan) m.t_global_scan += elapsed(pr.first, pr.second);
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
  if (m.local) {
    // the rows still live (their components froze in the last rounds) join the
    // parked ones: together they are this rank's input to the global phase
    RankState& R = L.ranks[0];
    RoundCounters rc;
    KDB_CUDA(cudaMemcpy(&rc, R.ctr, sizeof(rc), cudaMemcpyDeviceToHost));
    const uint32_t n_live = rc.na[cur];
    if (n_live)
      KDB_CUDA(cudaMemcpyAsync(R.park + hc.n_park, R.act[cur], n_live * sizeof(Rec), cudaMemcpyDeviceToDevice, st));
    m.n_park = hc.n_park + n_live;
    m.msf_local = hc.msf_count;
  }
  return KDB_OK;
}

// ---------------------------------------------------------------------------
// Local-first contraction (multi-rank exact mode, SURVEY.md
// §8(e)(ii)): the paper's local/cut split (Alg. 2 + Alg. 4, PAPER.md:538-541,
// 698-751) made exact.
//  1. Local phase, per rank, no exchange: rows-Boruvka on the rank's own rows
//     with LOCAL component ids.  A component hooks only along its certified
//     minimum when that minimum is a local edge -- the cut property makes every
//     such edge an MSF edge whatever the other ranks hold.  A component whose
//     minimum leaves the rank (or cannot be certified from its rows) freezes:
//     it never hooks again in this phase, and its rows are parked with their
//     heads.  Local components may still hook INTO it (its minimum then stays
//     the same edge).
//  2. Transition: global dense ids = rank offset + local id; the component ids
//     of every row, and the per-component minimum core id and certificate
//     bound, are all-gathered once (NCCL broadcasts, one per rank).
//  3. Global phase: the replicated-rounds Boruvka continues from the parked
//     rows over the components the local phases left (C_G).
// The forest is the Kruskal forest either way (every hook is a true minimum).
kdb_status local_first(Mst& m, float eps_run) {
  Layout& L = m.L;
  cudaStream_t st = m.st;
  kdb_comm* comm = m.comm;
  const bool nccl = multi_rank(comm);
  const int nr = (int)L.ranks.size();
  const int P = nccl ? comm->nranks : nr;
  const int me = nccl ? comm->rank : 0;  // first rank index this process runs
  cudaEvent_t* ev = m.ev;
  KDB_CUDA(cudaEventRecord(ev[3], st));
  // ---- every rank's rows --------------------------------------------------------
  int64_t* scratch = reinterpret_cast<int64_t*>(L.buckets);  // 256 x 8 B, free until the finalize
  if (P > 64) return set_err(KDB_EINVAL, "local-first phase supports at most 64 ranks");
  std::vector<int64_t> rb(P), rn(P);
  if (nccl) {
    int64_t h[2] = {L.ranks[0].row_begin, L.ranks[0].n_rows};
    KDB_CUDA(cudaMemcpyAsync(scratch + 2 * me, h, sizeof(h), cudaMemcpyHostToDevice, st));
    KDB_TRY(nccl_check(g_nccl.AllGather(scratch + 2 * me, scratch, 2, ncclInt64, comm->nccl, st), "ncclAllGather(rows)"));
    std::vector<int64_t> hh(2 * P);
    KDB_CUDA(cudaMemcpyAsync(hh.data(), scratch, 2 * P * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < P; ++r) { rb[r] = hh[2 * r]; rn[r] = hh[2 * r + 1]; }
  } else {
    for (int r = 0; r < P; ++r) { rb[r] = L.ranks[r].row_begin; rn[r] = L.ranks[r].n_rows; }
  }
  // global dense id of each rank's first core row, and its core-row count
  std::vector<int64_t> lo(P), C0(P);
  {
    std::vector<int64_t> pos(2 * P);
    for (int r = 0; r < P; ++r) { pos[2 * r] = rb[r]; pos[2 * r + 1] = rb[r] + rn[r]; }
    KDB_CUDA(cudaMemcpyAsync(scratch, pos.data(), 2 * P * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    LAUNCH(k_core_below, 1, 128, st, m.bits, L.woff, scratch, 2 * P, scratch + 2 * P);
    KDB_CUDA(cudaGetLastError());
    std::vector<int64_t> cnt(2 * P);
    KDB_CUDA(cudaMemcpyAsync(cnt.data(), scratch + 2 * P, 2 * P * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < P; ++r) { lo[r] = cnt[2 * r]; C0[r] = cnt[2 * r + 1] - cnt[2 * r]; }
  }
  // ---- 1. local phases ------------------------------------------------------------
  std::vector<int64_t> CL(P, 0), EC(P, 0), NP(P, 0);
  m.t_local_max = m.t_local_sum = 0;
  for (int ri = 0; ri < nr; ++ri) {
    const int r = me + ri;
    RankState& R = L.ranks[ri];
    if (C0[r] == 0) {  // no core row: nothing to contract, nothing to park
      R.compact = true;
      R.n_deep = 0;
      continue;
    }
    const int64_t o = lo[r];
    LAUNCH(k_shift_comp, grid_for(rn[r]), kThreads, st, m.comp + rb[r], rn[r], (int32_t)-o);
    Mst sub;
    sub.g = m.g;
    sub.comm = nullptr;
    sub.st = st;
    sub.N = m.N;
    sub.k = m.k;
    sub.ld = m.ld;
    sub.bits = m.bits;
    sub.comp = m.comp;
    sub.general = false;
    sub.local = true;
    sub.lv.lo = rb[r];
    sub.lv.hi = rb[r] + rn[r];
    sub.lv.bits = m.bits;
    sub.C0 = C0[r];
    sub.ecap = C0[r];
    for (int i = 0; i < 4; ++i) sub.ev[i] = m.ev[i];
    Layout& S = sub.L;
    S = L;
    S.cmin += o; S.cmin2 += o; S.parent += o; S.rootof += o; S.newid += o; S.flag += o;
    S.kmin += o; S.kmin2 += o; S.Kc += o; S.Bc += o; S.tgt += o; S.e_key += o; S.e_w += o;
    S.rec1 += o; S.frz += o; S.frz2 += o;
    S.ctr = R.lctr;
    S.ranks.assign(1, R);
    S.ranks[0].Kc = S.Kc;
    S.ranks[0].Bc = S.Bc;
    S.ranks[0].tgt = S.tgt;
    KDB_TRY(rows_phase(sub, eps_run));
    R.n_deep = sub.L.ranks[0].n_deep;
    R.n_local = sub.L.ranks[0].n_local;
    R.compact = sub.L.ranks[0].compact;
    CL[r] = sub.C;
    EC[r] = (int64_t)sub.msf_local;
    NP[r] = (int64_t)sub.n_park;
    const double t = sub.t_init + sub.t_min_edges;
    m.t_local_max = std::max(m.t_local_max, t);
    m.t_local_sum += t;
    m.entries += sub.entries;
    m.rounds = std::max(m.rounds, sub.rounds);
    m.local_rounds = std::max(m.local_rounds, sub.rounds);
  }
  KDB_CUDA(cudaEventRecord(ev[1], st));
  // ---- 2. transition -----------------------------------------------------------------
  if (nccl) {  // every rank's (components, local MSF edges, parked rows)
    int64_t h[3] = {CL[me], EC[me], NP[me]};
    KDB_CUDA(cudaMemcpyAsync(scratch + 3 * me, h, sizeof(h), cudaMemcpyHostToDevice, st));
    KDB_TRY(nccl_check(g_nccl.AllGather(scratch + 3 * me, scratch, 3, ncclInt64, comm->nccl, st), "ncclAllGather(counts)"));
    std::vector<int64_t> hh(3 * P);
    KDB_CUDA(cudaMemcpyAsync(hh.data(), scratch, 3 * P * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < P; ++r) { CL[r] = hh[3 * r]; EC[r] = hh[3 * r + 1]; NP[r] = hh[3 * r + 2]; }
  }
  std::vector<int64_t> off(P + 1, 0), eoff(P + 1, 0);
  for (int r = 0; r < P; ++r) { off[r + 1] = off[r] + CL[r]; eoff[r + 1] = eoff[r] + EC[r]; }
  const int64_t CG = off[P];
  // this process's ranks: per-component data to the global dense positions
  // (into the *2 arrays, swapped below), row ids local -> global, local MSF
  // edges compacted (sim: all ranks in rank order; NCCL: this rank's at 0)
  uint64_t* tK = L.Kc;                              // free: refilled for the global phase
  uint32_t* tA = reinterpret_cast<uint32_t*>(L.Bc);  // e_w holds the a endpoint as u32
  int64_t e_here = 0;
  for (int ri = 0; ri < nr; ++ri) {
    const int r = me + ri;
    if (C0[r] == 0) continue;
    if (CL[r] > 0) {
      KDB_CUDA(cudaMemcpyAsync(L.cmin2 + off[r], L.cmin + lo[r], CL[r] * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
      KDB_CUDA(cudaMemcpyAsync(L.kmin2 + off[r], L.kmin + lo[r], CL[r] * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    }
    LAUNCH(k_shift_comp, grid_for(rn[r]), kThreads, st, m.comp + rb[r], rn[r], (int32_t)off[r]);
    const int64_t eo = nccl ? 0 : eoff[r];
    if (EC[r] > 0) {
      KDB_CUDA(cudaMemcpyAsync(tK + eo, L.e_key + lo[r], EC[r] * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
      KDB_CUDA(cudaMemcpyAsync(tA + eo, reinterpret_cast<const uint32_t*>(L.e_w) + lo[r], EC[r] * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice, st));
    }
    e_here += EC[r];
  }
  KDB_CUDA(cudaGetLastError());
  if (nccl) {  // replicate: every rank's row ids and its components' (cmin, kmin)
    KDB_TRY(nccl_check(g_nccl.GroupStart(), "ncclGroupStart"));
    for (int r = 0; r < P; ++r) {
      if (rn[r] > 0)
        KDB_TRY(nccl_check(g_nccl.Broadcast(m.comp + rb[r], m.comp + rb[r], (size_t)rn[r], ncclInt32, r, comm->nccl, st),
                           "ncclBroadcast(comp)"));
      if (CL[r] > 0) {
        KDB_TRY(nccl_check(g_nccl.Broadcast(L.cmin2 + off[r], L.cmin2 + off[r], (size_t)CL[r], ncclInt32, r,
                                            comm->nccl, st), "ncclBroadcast(cmin)"));
        KDB_TRY(nccl_check(g_nccl.Broadcast(L.kmin2 + off[r], L.kmin2 + off[r], (size_t)CL[r], ncclUint32, r,
                                            comm->nccl, st), "ncclBroadcast(kmin)"));
      }
    }
    KDB_TRY(nccl_check(g_nccl.GroupEnd(), "ncclGroupEnd"));
  }
  m.payload_transition = 4.0 * (double)m.N + 8.0 * (double)CG;
  std::swap(L.cmin, L.cmin2);
  std::swap(L.kmin, L.kmin2);
  std::swap(L.e_key, L.Kc);
  {
    float* w = L.e_w;
    L.e_w = reinterpret_cast<float*>(L.Bc);
    L.Bc = reinterpret_cast<uint32_t*>(w);
  }
  L.ranks[0].Kc = L.Kc;
  L.ranks[0].Bc = L.Bc;
  // ---- 3. global phase ---------------------------------------------------------------
  KDB_CUDA(cudaMemsetAsync(L.ctr, 0, sizeof(RoundCounters), st));
  {
    const uint32_t ec = (uint32_t)e_here;
    KDB_CUDA(cudaMemcpyAsync(&L.ctr->msf_count, &ec, sizeof(ec), cudaMemcpyHostToDevice, st));
  }
  uint64_t parked = 0;
  for (int r = 0; r < P; ++r) parked += (uint64_t)NP[r];
  for (int ri = 0; ri < nr; ++ri) {
    const int r = me + ri;
    RankState& R = L.ranks[ri];
    KDB_CUDA(cudaMemsetAsync(R.ctr, 0, sizeof(RoundCounters), st));
    const uint32_t np = (uint32_t)NP[r];
    if (np) KDB_CUDA(cudaMemcpyAsync(R.act[0], R.park, np * sizeof(Rec), cudaMemcpyDeviceToDevice, st));
    KDB_CUDA(cudaMemcpyAsync(&R.ctr->na[0], &np, sizeof(np), cudaMemcpyHostToDevice, st));
    R.n_act = np;
    R.n_in_act = 0;
    if (!R.compact && R.n_rows > 0) return set_err(KDB_EINTERNAL, "local-first phase without the light ELL");
  }
  for (int ri = 0; ri < nr; ++ri)
    if (CG > 0) LAUNCH(k_fill_comp_arrays, grid_for(CG), kThreads, st, CG, L.ranks[ri].Kc, L.ranks[ri].Bc, nullptr);
  KDB_CUDA(cudaGetLastError());
  KDB_CUDA(cudaEventRecord(ev[2], st));
  m.t_transition = elapsed(ev[1], ev[2]);
  m.t_init += elapsed(ev[3], ev[2]) - m.t_transition;  // local phases (all virtual ranks, in sequence)
  m.C_global = CG;
  m.parked_rows = parked;
  m.cont = true;
  m.C = CG;
  const double tmin0 = m.t_min_edges;
  KDB_TRY(rows_phase(m, eps_run));
  m.cont = false;
  m.t_global = m.t_min_edges - tmin0;
  return KDB_OK;
}

// Filter: every rank streams its rows once and keeps the heavy candidate
// entries (tau < w <= eps) whose endpoints lie in different light components.
kdb_status filter_phase(Mst& m, float eps, bool* overflow) {
  Layout& L = m.L;
  cudaStream_t st = m.st;
  KDB_CUDA(cudaEventRecord(m.ev[0], st));
  // KDB_SURVCAP (tests): a smaller survivor capacity, to exercise the fallback
  const int64_t cap_env = opt_int("KDB_SURVCAP", -1);
  // fast-path tables (identical on every rank: comp is replicated)
  int shift = 0;
  while (((m.N + ((int64_t)1 << shift) - 1) >> shift) > kDomMax) ++shift;
  const int64_t nblk = (m.N + ((int64_t)1 << shift) - 1) >> shift;
  bool fast = opt_int("KDB_FASTFILTER", 1) != 0;
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
    // per-block runs (host: nblk <= kDomMax): a component whose dominated blocks
    // are not ONE contiguous run has no range in rng (its ids come in several
    // runs, e.g. a cluster split by the data set's partition); its
    // rows then use the run of equal-dom blocks around their own block
    std::vector<int32_t> hdom(nblk);
    std::vector<int2> hrun(nblk);
    KDB_CUDA(cudaMemcpyAsync(hdom.data(), L.dom, nblk * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaMemcpyAsync(fc, L.fcount, sizeof(fc), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    for (int64_t b = 0; b < nblk;) {
      int64_t e = b + 1;
      while (e < nblk && hdom[e] == hdom[b]) ++e;
      const int2 r = hdom[b] >= 0 ? make_int2((int32_t)(b << shift), (int32_t)std::min<int64_t>(e << shift, m.N))
                                  : make_int2(1, 0);
      for (int64_t x = b; x < e; ++x) hrun[x] = r;
      b = e;
    }
    KDB_CUDA(cudaMemcpyAsync(L.brun, hrun.data(), nblk * sizeof(int2), cudaMemcpyHostToDevice, st));
    KDB_CUDA(cudaStreamSynchronize(st));  // hrun is a host temporary
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
    // umulhi(n, m32) == n / d for n * d < 2^32; tile indices n < kFilterRows * d
    fd.small = (fd.d > 1 && fd.d * fd.d * (uint64_t)kFilterRows < (1ull << 32)) ? 1u : 0u;
    const int64_t ntiles = (R.n_rows + kFilterRows - 1) / kFilterRows;  // warp tiles
    const int grid = (int)std::min<int64_t>((ntiles + kFilterWarps - 1) / kFilterWarps, 1 << 30);
#define KDB_FILTER_LAUNCH2(V, F, CO, SM)                                                                         \
  LAUNCH_DYN((k_filter<V, F, CO, SM>), grid, kFilterThreads, kFilterSmem, st, R.nbr, R.dist, R.n_rows, m.ld, m.k,  \
             m.tau, eps, R.row_begin, m.N, m.comp, rng, L.bloom, fd, R.hs[0], R.hs_cap, R.n_hs_dev, L.fcount + 1, \
             L.dom, L.brun, shift)
  // the row-within-tile division: a 32-bit multiply-high when exact (compile-time
  // branch: it runs once per 16-B chunk of the sweep)
#define KDB_FILTER_LAUNCH(V, F, CO)                                                                              \
  do {                                                                                                           \
    if (fd.small) KDB_FILTER_LAUNCH2(V, F, CO, true);                                                          \
    else KDB_FILTER_LAUNCH2(V, F, CO, false);                                                                  \
  } while (0)
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
#undef KDB_FILTER_LAUNCH2
    KDB_CUDA(cudaGetLastError());
  }
  uint32_t over = 0;
  unsigned long long tot = 0;
  for (auto& R : L.ranks) {
    uint32_t nf[2] = {0, 0};  // count, sticky overflow flag
    KDB_CUDA(cudaMemcpyAsync(nf, R.n_hs_dev, 8, cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    R.n_hs = nf[0];
    tot += nf[0];
    if (nf[0] > R.hs_cap || nf[1]) over = 1;
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
  // per-round spans (events, read after the round's host sync): A = per-rank
  // work (fills of ranks >= 1, offers, compaction), B = sim reductions, C = per-rank ties
  cudaEvent_t hv[7];
  for (auto& e : hv) KDB_CUDA(cudaEventCreate(&e));
  struct HvGuard { cudaEvent_t* e; ~HvGuard() { for (int i = 0; i < 7; ++i) cudaEventDestroy(e[i]); } } hvg{hv};
  while (C > 1) {
    ++rounds;
    LAUNCH(k_fill_comp_arrays, grid_for(C), kThreads, st, C, L.Kc, L.Bc, nullptr);
    KDB_CUDA(cudaEventRecord(hv[0], st));
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
    KDB_CUDA(cudaEventRecord(hv[1], st));
    KDB_CUDA(cudaStreamSynchronize(st));
    m.t_heavy_rank += elapsed(hv[0], hv[1]);
    KDB_CUDA(cudaEventRecord(hv[2], st));
    for (size_t r = 1; r < L.ranks.size(); ++r)
      LAUNCH(k_min_into_u64, grid_for(C), kThreads, st, L.Kc, L.ranks[r].Kc, C);
    KDB_CUDA(cudaEventRecord(hv[3], st));
    KDB_TRY(allreduce_min_u64(comm, L.Kc, C, st));
    m.payload_heavy += 8.0 * C;
    KDB_CUDA(cudaEventRecord(hv[4], st));
    for (size_t r = 0; r < L.ranks.size(); ++r) {
      RankState& R = L.ranks[r];
      if (R.n_hs)
        LAUNCH(k_hedge_tie, grid_for(R.n_hs), kThreads, st, R.hs[cur[r]], R.n_hs, L.hcomp, L.Kc, R.Bc);
    }
    KDB_CUDA(cudaEventRecord(hv[5], st));
    for (size_t r = 1; r < L.ranks.size(); ++r)
      LAUNCH(k_min_into_u32, grid_for(C), kThreads, st, L.Bc, L.ranks[r].Bc, C);
    KDB_CUDA(cudaEventRecord(hv[6], st));
    KDB_TRY(allreduce_min_u32(comm, L.Bc, C, st));
    m.payload_heavy += 4.0 * C;
    KDB_CUDA(cudaMemsetAsync(&L.ctr->hooks, 0, 4 * sizeof(uint32_t), st));
    LAUNCH(k_hook_h, grid_for(C), kThreads, st, C, L.Kc, L.Bc, m.comp, L.hcomp, L.parent, L.e_key, L.e_w, m.N, L.ctr);
    KDB_CUDA(cudaGetLastError());
    RoundCounters hc;
    KDB_CUDA(cudaMemcpyAsync(&hc, L.ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
    KDB_CUDA(cudaStreamSynchronize(st));
    m.t_heavy_simred += elapsed(hv[2], hv[3]) + elapsed(hv[5], hv[6]);
    m.t_heavy_rank += elapsed(hv[4], hv[5]);
    if (hc.offered == 0) break;
    if (hc.hooks == 0) return set_err(KDB_EINTERNAL, "heavy phase made no progress");
    LAUNCH(k_jump, grid_for(C), kThreads, st, C, L.parent, L.rootof, L.ctr, (const int64_t*)nullptr, L.flag);
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

