// kdb_oracle.cpp -- the CPU ORACLE for the kNN-DBSCAN clustering stage.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  The product
// path (paper_2009_04552_b200/) never links, imports or calls it, and this file
// shares no code, header or constant generator with the CUDA path.
//
// What it computes: the exactly-defined result the paper's method reaches
// (Thm. 2: clusters of core points = components of the MST
// of the core-core graph; Thm. 3: any partitioning gives the
// same clusters), written out as its plain definition:
//
//   1. core[i]   = D[i][M-1] <= eps                      Alg. 1 line 4,
//                                                         Lemma 1(i)
//   2. candidate edges: every stored entry (i, c) with J = nbr[i][c] >= 0, J != i,
//      core[i], core[J], D[i][c] <= eps becomes the undirected edge {i, J} with
//      weight w = D[i][c] and key (mono(w), a = min(i,J), b = max(i,J)).
//      Both directed copies are kept (they coincide when weights are symmetric).
//      -- north_star "core-core kNN edges with weight <= eps"; reading #3/#4.
//   3. MSF: sort by key, Kruskal with union-find; accept iff endpoints are in
//      different sets.  Output sorted by (a, b); total weight = fp64 sum of the
//      accepted weights in key order.           -- Def. 10 / Thm. 2
//   4. label of a core point = minimum core index of its tree (union by min index).
//                                               -- north_star "canonical labels"
//   5. border: for non-core i, the first entry in stored row order with J >= 0,
//      core[J] and D[i][c] <= eps gives label[i] = label[J]; none -> -1 (noise).
//                                               -- Lemma 1(ii),
//                                                  SPEC.md:344, reading #13
//
// edge_cols: candidate entries are taken from the first
// edge_cols columns of each row only.  edge_cols = k is the all-k reading #3
// (north_star); edge_cols = M is the paper's own kNN-DBSCAN edge set -- direct
// M-reachability, Def. 6: q in N_M(p) or p in N_M(q), and
// Alg. 2's scan bound L[i] <= M; Thm. 2(ii):
// the MST clusters of G_M,core are the kNN-DBSCAN clusters.
//
// Pins (tests/test_oracle_pins.py): worked examples W1-W3 from the paper's
// Fig. cycle / Fig. cut_mst (tests/golden/), brute-force classic DBSCAN at
// k = N-1 (Thm. 2(i)), Prim's MSF weight multiset, brute-force MSF enumeration,
// BFS components, the cycle-property certificate, Thm. 1 containment and the
// brute-force nearest-core border rule.
//
// Build: g++ -O2 -std=c++17 -shared -fPIC (see Makefile).

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

// mono(w): the fp32 bit pattern of a non-negative weight, -0 canonicalised to +0.
// For non-negative IEEE floats the bit pattern orders like the value.
inline uint32_t mono(float w) {
  uint32_t u;
  std::memcpy(&u, &w, 4);
  if (u == 0x80000000u) u = 0u;
  return u;
}

struct Edge {
  uint32_t mw;  // mono(w)
  uint32_t a;   // min endpoint
  uint32_t b;   // max endpoint
  float w;
};

inline bool key_less(const Edge& x, const Edge& y) {
  if (x.mw != y.mw) return x.mw < y.mw;
  if (x.a != y.a) return x.a < y.a;
  return x.b < y.b;
}

// union-find with union by minimum index: the root of every set is its
// smallest member, so find(i) is the canonical label directly.
struct DSU {
  std::vector<uint32_t> p;
  explicit DSU(int64_t n) : p((size_t)n) {
    for (int64_t i = 0; i < n; ++i) p[(size_t)i] = (uint32_t)i;
  }
  uint32_t find(uint32_t x) {
    while (p[x] != x) {
      p[x] = p[p[x]];
      x = p[x];
    }
    return x;
  }
  bool unite(uint32_t x, uint32_t y) {
    x = find(x);
    y = find(y);
    if (x == y) return false;
    if (x < y) p[y] = x; else p[x] = y;
    return true;
  }
};

double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

// Step 1. core[i] = (dist[i*k + M-1] <= eps).  Returns 0, or -1 on bad args.
int oracle_core_mark(int64_t n, int32_t k, const float* dist, int32_t M, float eps,
                     uint8_t* core) {
  if (n < 0 || k < 1 || M < 1 || M > k) return -1;
  for (int64_t i = 0; i < n; ++i) core[i] = (dist[i * (int64_t)k + (M - 1)] <= eps) ? 1 : 0;
  return 0;
}

// Step 2. Number of candidate entries (directed copies counted separately) in
// the first edge_cols columns.
int64_t oracle_candidate_count(int64_t n, int32_t k, const int32_t* nbr, const float* dist,
                               const uint8_t* core, float eps, int32_t edge_cols) {
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!core[i]) continue;
    for (int32_t c = 0; c < edge_cols; ++c) {
      int64_t J = nbr[i * (int64_t)k + c];
      float w = dist[i * (int64_t)k + c];
      if (J >= 0 && J < n && J != i && core[J] && w <= eps) ++m;
    }
  }
  return m;
}

// Step 2 (materialised): the candidate multiset in row order as (a, b, w).
int64_t oracle_candidates(int64_t n, int32_t k, const int32_t* nbr, const float* dist,
                          const uint8_t* core, float eps, int32_t edge_cols, uint32_t* ea, uint32_t* eb,
                          float* ew, int64_t cap) {
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!core[i]) continue;
    for (int32_t c = 0; c < edge_cols; ++c) {
      int64_t J = nbr[i * (int64_t)k + c];
      float w = dist[i * (int64_t)k + c];
      if (J >= 0 && J < n && J != i && core[J] && w <= eps) {
        if (m < cap) {
          ea[m] = (uint32_t)std::min<int64_t>(i, J);
          eb[m] = (uint32_t)std::max<int64_t>(i, J);
          ew[m] = w;
        }
        ++m;
      }
    }
  }
  return m;
}

// Steps 3-4 on an explicit undirected multigraph (a[e], b[e], w[e]) over n
// vertices: Kruskal under key (mono(w), min, max).  Writes comp[v] = min index of
// v's tree for v with is_vertex[v] (others -1), the accepted edges sorted by
// (a, b), their count and their fp64 weight sum (in key order).
int oracle_kruskal(int64_t n, int64_t m, const uint32_t* ea, const uint32_t* eb, const float* ew,
                   const uint8_t* is_vertex, int32_t* comp, uint32_t* ma, uint32_t* mb,
                   float* mw, int64_t cap, int64_t* count, double* weight) {
  std::vector<Edge> E((size_t)m);
  for (int64_t e = 0; e < m; ++e) {
    uint32_t a = std::min(ea[e], eb[e]), b = std::max(ea[e], eb[e]);
    E[(size_t)e] = Edge{mono(ew[e]), a, b, ew[e]};
  }
  std::sort(E.begin(), E.end(), key_less);
  DSU dsu(n);
  std::vector<Edge> T;
  double total = 0.0;
  for (const Edge& e : E) {
    if (dsu.unite(e.a, e.b)) {
      T.push_back(e);
      total += (double)e.w;
    }
  }
  std::sort(T.begin(), T.end(), [](const Edge& x, const Edge& y) {
    return x.a != y.a ? x.a < y.a : x.b < y.b;
  });
  if ((int64_t)T.size() > cap) return -2;
  for (size_t t = 0; t < T.size(); ++t) {
    ma[t] = T[t].a;
    mb[t] = T[t].b;
    mw[t] = T[t].w;
  }
  *count = (int64_t)T.size();
  *weight = total;
  for (int64_t v = 0; v < n; ++v) comp[v] = is_vertex[v] ? (int32_t)dsu.find((uint32_t)v) : -1;
  return 0;
}

// Step 5. labels[i] = comp[i] for core i; for non-core i the first entry in
// stored order with J >= 0, core[J], D <= eps gives comp[J]; else -1.
int oracle_border(int64_t n, int32_t k, const int32_t* nbr, const float* dist,
                  const uint8_t* core, float eps, const int32_t* comp, int32_t* labels) {
  for (int64_t i = 0; i < n; ++i) {
    if (core[i]) {
      labels[i] = comp[i];
      continue;
    }
    labels[i] = -1;
    for (int32_t c = 0; c < k; ++c) {
      int64_t J = nbr[i * (int64_t)k + c];
      float w = dist[i * (int64_t)k + c];
      if (J >= 0 && J < n && core[J] && w <= eps) {
        labels[i] = comp[J];
        break;
      }
    }
  }
  return 0;
}

// The whole stage (Alg. 1, as its plain definition).
// times[0..2] = seconds spent in core / candidates+Kruskal / border.
// Returns 0; -1 bad args; -2 msf_cap too small.
int oracle_kdbscan(int64_t n, int32_t k, const int32_t* nbr, const float* dist, int32_t M,
                   float eps, int32_t edge_cols, uint8_t* core, int32_t* labels, uint32_t* msf_a,
                   uint32_t* msf_b, float* msf_w, int64_t msf_cap, int64_t* msf_count,
                   double* msf_weight, double* times) {
  if (n < 0 || k < 1 || M < 1 || M > k || !(eps > 0.0f) || edge_cols < 1 || edge_cols > k) return -1;
  double t0 = now_s();
  oracle_core_mark(n, k, dist, M, eps, core);
  double t1 = now_s();
  int64_t m = oracle_candidate_count(n, k, nbr, dist, core, eps, edge_cols);
  std::vector<uint32_t> ea((size_t)m), eb((size_t)m);
  std::vector<float> ew((size_t)m);
  oracle_candidates(n, k, nbr, dist, core, eps, edge_cols, ea.data(), eb.data(), ew.data(), m);
  std::vector<int32_t> comp((size_t)n);
  int rc = oracle_kruskal(n, m, ea.data(), eb.data(), ew.data(), core, comp.data(), msf_a, msf_b,
                          msf_w, msf_cap, msf_count, msf_weight);
  if (rc) return rc;
  double t2 = now_s();
  oracle_border(n, k, nbr, dist, core, eps, comp.data(), labels);
  double t3 = now_s();
  if (times) {
    times[0] = t1 - t0;
    times[1] = t2 - t1;
    times[2] = t3 - t2;
  }
  return 0;
}

}  // extern "C"
