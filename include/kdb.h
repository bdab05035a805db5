/* kdb.h -- C-ABI of the B200-native kNN-DBSCAN clustering stage.
 *
 * The stage (Alg. 1 "Parallel kNN-DBSCAN") takes a directed
 * k-nearest-neighbour graph G_k of N points (k >= M) split into contiguous row
 * ranges over p processes ("we partition points evenly into each
 * process"), a radius eps and a minimum neighbourhood size M, and returns
 *   - core flags            (Alg. 1 lines 3-8; Lemma 1(i)),
 *   - the exact minimum spanning forest of the core-core candidate edges
 *     (Alg. 2/3 Boruvka; Def. 10 / Thm. 2),
 *   - canonical labels: the minimum core index of a point's component, -1 noise
 *     (north_star; border rule = Lemma 1(ii), "ClusterBorder" PAPER.md:543).
 *
 * Graph convention (SURVEY.md §8(c) readings #1, #17-#19):
 *   row i lists i's neighbours EXCLUDING i itself, weights non-decreasing fp32,
 *   padding entries are (id -1, weight +inf) at the row tail.  core(i) is
 *   D[i][M-1] <= eps, i.e. at least M other points within eps.
 * Candidate edges: every stored entry (i, c) with c < edge_cols, J = nbr[i][c] >= 0,
 *   J != i, core(i), core(J) and D[i][c] <= eps is the UNDIRECTED edge {i, J}
 *   with weight w = D[i][c] (reading #4: undirected).  edge_cols = k (the
 *   default) is reading #3, all k columns; edge_cols = M is the paper's direct
 *   M-reachability, Def. 6: p core and q in N_M(p) or
 *   p in N_M(q), with Alg. 2's scan bound L[i] <= M; by
 *   Thm. 2(ii) its MSF clusters are the kNN-DBSCAN clusters.
 * Edge order O1 (reading #6): (mono(w), a = min(i,J), b = max(i,J)) where
 *   mono(w) is the fp32 bit pattern with -0 canonicalised to +0.  The MSF under
 *   this strict order is unique; kdb_mst returns exactly it.
 *
 * Conventions for every call:
 *   - All array arguments are DEVICE pointers owned by the caller (the library
 *     never allocates device memory outside `workspace` and keeps no global
 *     device state).  Host pointers are marked "host".
 *   - Work is ordered on `stream` (a cudaStream_t).  kdb_core_mark and kdb_label
 *     are asynchronous; kdb_mst synchronises `stream` (one small read-back per
 *     Boruvka round) and returns host scalars.
 *   - Host-side argument validation runs before any launch; on failure nothing
 *     is launched and KDB_EINVAL is returned.  kdb_last_error() gives a
 *     thread-local message for the most recent non-OK status.
 *   - Multi-GPU: every rank calls with the same N, M, eps and a communicator;
 *     rank r passes its own rows [row_begin, row_begin + n_rows).  Outputs that
 *     are documented as replicated are identical on every rank.
 */
#ifndef KDB_H_
#define KDB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KDB_OK = 0,
  KDB_EINVAL = 1,    /* invalid argument (see each call)                         */
  KDB_ENOMEM = 2,    /* workspace smaller than kdb_mst_workspace_bytes()         */
  KDB_ECUDA = 3,     /* CUDA runtime error; message in kdb_last_error()          */
  KDB_ENCCL = 4,     /* NCCL error / NCCL library not loadable                   */
  KDB_EINTERNAL = 5  /* internal invariant violated (a bug); message attached    */
} kdb_status;

typedef struct CUstream_st* kdb_stream_t; /* == cudaStream_t */

/* Caller promise: the graph is an EXACT kNN graph of a point set under a
 * symmetric distance (rows hold each point's k nearest other points; every
 * weight is d(i,J) computed identically from both ends).  Under this promise
 * an entry u->v that v's row does not mirror has w >= D[v][k-1],
 * which lets kdb_mst skip building reverse-edge lists.  Without it kdb_mst
 * materialises in-edge lists in the workspace (correct for ANY valid graph,
 * e.g. the approximate graph of Fig. cycle). */
#define KDB_GRAPH_EXACT 1u

/* Caller promise for an eps sweep (Fig. eps_mnist protocol, PAPER.md:459-488:
 * one kNN graph, many eps): this kdb_mst call gets the same graph (pointers,
 * contents, row range, k_max, edge_cols) and the same workspace as the
 * previous kdb_mst call on that workspace, and nothing else wrote the
 * workspace in between -- only eps and core_bits differ.  The library may then
 * reuse the light ELL it built from the graph (the first 16 entries of every row
 * and each row's certificate bound: they depend on the graph and the light
 * threshold, the median of a fixed column, not on eps).  It checks the pointers,
 * sizes and threshold it recorded for that workspace and rebuilds on any
 * mismatch; the contents are the caller's promise.  One process / one rank
 * only (ignored otherwise).  Results are identical either way. */
#define KDB_GRAPH_REUSE 2u

typedef struct {
  int64_t n_total;     /* N = |I|, all ranks                                        */
  int64_t row_begin;   /* first global row id held by this rank                     */
  int64_t n_rows;      /* rows held by this rank; [row_begin, row_begin+n_rows) in [0,N) */
  int32_t k_max;       /* row stride k, 1 <= k <= 65535                             */
  const int32_t* nbr;  /* device [n_rows][k_max] global ids, -1 = padding; 16-B aligned */
  const float* dist;   /* device [n_rows][k_max] fp32 >= 0, non-decreasing per row,
                          +inf = padding; 16-B aligned                              */
  uint32_t flags;      /* KDB_GRAPH_EXACT and/or KDB_GRAPH_REUSE, or 0                */
  int32_t edge_cols;   /* candidate edges come from columns [0, edge_cols) of each row;
                          0 = all k_max.  Only kdb_mst reads it; 0 <= edge_cols <= k_max
                          (EINVAL otherwise).  edge_cols = M gives Def. 6's edge set.
                          The kernels keep the row stride k_max and never read columns
                          >= edge_cols (the first edge_cols columns of an exact k-NN
                          graph are an exact edge_cols-NN graph, so KDB_GRAPH_EXACT
                          stays valid with the certificate taken at column edge_cols-1). */
} kdb_graph;

/* ---- communicators ------------------------------------------------------ */
typedef struct kdb_comm kdb_comm; /* NULL => single GPU, this process owns all rows */

/* NCCL backend over NVLink/NVSwitch.  `nccl_unique_id` is the 128-byte
 * ncclUniqueId produced by kdb_nccl_unique_id() on rank 0 and broadcast by the
 * caller (e.g. torch.distributed).  Each rank must have selected its device.
 * The NCCL shared library is dlopen()ed from $KDB_NCCL_LIBRARY, else
 * "libnccl.so.2". */
kdb_status kdb_nccl_unique_id(void* out_128_bytes /* host */);
kdb_status kdb_comm_create_nccl(kdb_comm** out, const void* nccl_unique_id /* host, 128 B */,
                                int rank, int nranks);
/* Single-GPU simulation of `nranks` ranks (tests): the caller passes the FULL
 * graph (row_begin 0, n_rows N); the library splits rows into nranks
 * contiguous ranges, keeps per-virtual-rank partial results and reduces them
 * exactly as the NCCL backend would.  Results must equal the NULL-comm run. */
kdb_status kdb_comm_create_sim(kdb_comm** out, int nranks);
void kdb_comm_destroy(kdb_comm* comm);

/* ---- the three calls of Alg. 1 ------------------------------------------ */

/* Alg. 1 lines 3-8, Lemma 1(i):
 *   core(v) = dist[v][M-1] <= eps   for this rank's rows v.
 * core_bits: device uint32[ceil(N/32)], bit (v & 31) of word v >> 5.  The call
 * zeroes it, sets the bits of local rows and, with a communicator, combines all
 * ranks' bits so every rank ends with all N flags (replicated).
 * EINVAL: M < 1 or M > k_max, eps not in (0, +inf), null pointers, bad ranges. */
kdb_status kdb_core_mark(const kdb_graph* g, int32_t M, float eps, uint32_t* core_bits,
                         kdb_comm* comm, kdb_stream_t stream);

/* Bytes of device workspace kdb_mst needs for this graph (depends on N,
 * n_rows, k_max, flags and the communicator's rank count). */
size_t kdb_mst_workspace_bytes(const kdb_graph* g, kdb_comm* comm);

/* Alg. 1 lines 10-12: ParallelLocalMST + DistributedCutMST,
 * realised as exact Boruvka.  With more than one
 * rank and an exact graph (KDB_GRAPH_EXACT) every rank first contracts its own
 * rows without any exchange (the exact form of the paper's local MST: a
 * component hooks only along a certified minimum that stays inside the rank),
 * then the components left are finished by exchanged rounds.
 *   core_bits : device, replicated output of kdb_core_mark.
 *   comp      : device int32[N] out, replicated: for core v the minimum core id of
 *               v's component (the canonical label), -1 for non-core v.
 *   mst_a/b/w : device [mst_cap] out: the MSF edges {a < b} with weight w, sorted
 *               by (a, b).  One process: the whole forest.  A real multi-rank NCCL
 *               communicator: the edges whose smaller endpoint a lies in THIS
 *               rank's rows [row_begin, row_begin + n_rows) -- the ranks' outputs
 *               concatenated in rank order are the whole sorted forest.
 *               mst_cap >= #core - 1 suffices (EINVAL if the output does not fit).
 *   mst_count : host out, number of MSF edges returned (this rank's share).
 *   mst_weight: host out, the fp64 sum of the MSF weights, computed exactly and
 *               rounded once (independent of summation order and of the rank count).
 *   workspace : device, >= kdb_mst_workspace_bytes(g, comm) bytes, 256-B aligned.
 * Synchronises `stream`. */
kdb_status kdb_mst(const kdb_graph* g, float eps, const uint32_t* core_bits, int32_t* comp,
                   uint32_t* mst_a, uint32_t* mst_b, float* mst_w, int64_t mst_cap,
                   int64_t* mst_count, double* mst_weight, void* workspace, size_t ws_bytes,
                   kdb_comm* comm, kdb_stream_t stream);

/* The paper's INEXACT MST (PAPER.md:1053-1060,
 * Alg. 2 ParallelLocalMST + Alg. 4 DistributedCutMST):
 * vertex-partition the N points into `nparts` contiguous groups
 * [floor(pN/nparts), floor((p+1)N/nparts)) (the distributed row layout,
 * PAPER.md:517); MST_p,local = the MSF of group p's internal candidate edges;
 * every local subtree is a super vertex; MST_cut = the MSF of the candidate
 * edges between groups over the super vertices.  Output = U_p MST_p,local U
 * MST_cut, every MSF taken under O1 of the original edges.  By Thm. 3(ii)
 * comp/labels equal kdb_mst's; the forest and its weight in
 * general do not (weight >= kdb_mst's).  Arguments and outputs as kdb_mst;
 * single process (the whole graph: row_begin 0, n_rows = n_total), workspace
 * >= kdb_mst_inexact_workspace_bytes(g, nparts).  EINVAL: nparts < 1, a partial
 * graph, n_rows * edge_cols >= 2^31 - 1.  Synchronises `stream`. */
size_t kdb_mst_inexact_workspace_bytes(const kdb_graph* g, int32_t nparts);
kdb_status kdb_mst_inexact(const kdb_graph* g, float eps, const uint32_t* core_bits, int32_t nparts, int32_t* comp,
                           uint32_t* mst_a, uint32_t* mst_b, float* mst_w, int64_t mst_cap, int64_t* mst_count,
                           double* mst_weight, void* workspace, size_t ws_bytes, kdb_stream_t stream);

/* Alg. 1 line 13 ClusterBorder (body omitted in the paper,
 * SURVEY.md §8(c) reading #13, Lemma 1(ii)):
 *   labels[i] (device int32[n_rows]) for local row v = row_begin + i:
 *     core v     -> comp[v];
 *     non-core v -> comp[J] of the FIRST entry in stored row order with J >= 0,
 *                   core(J) and D <= eps (the scan stops at the first D > eps);
 *                   -1 (noise) if none.
 * Asynchronous. */
kdb_status kdb_label(const kdb_graph* g, float eps, const uint32_t* core_bits, const int32_t* comp,
                     int32_t* labels, kdb_stream_t stream);

/* Clustering quality.  The paper reports NMI
 * ("normalized mutual information ... almost one", PAPER.md:340,
 * 389) without a formula; the convention is SPEC.md:421-431:
 *   NMI(A, B) = 2 I(A;B) / (H(A) + H(B)), natural log, over the joint label
 *   histogram, every NOISE (-1) point in ONE shared pseudo-cluster per
 *   labelling; both entropies 0 -> 1; exactly one entropy 0 -> 0.
 *   clusters_a/_b: the number of distinct non-NOISE labels.
 * a, b: device int32[n] labels (>= -1; any values, e.g. kdb_label output and a
 * generator's ground truth).  nmi, clusters_a, clusters_b: host outputs.
 * workspace: device, >= kdb_nmi_workspace_bytes(n) bytes, 256-B aligned.
 * EINVAL: NULL pointers, n outside [0, 2^31-1), a label < -1.  ENOMEM: small
 * workspace.  Synchronises `stream`; n = 0 gives nmi = 1, no clusters. */
size_t kdb_nmi_workspace_bytes(int64_t n);
kdb_status kdb_nmi(const int32_t* a, const int32_t* b, int64_t n, double* nmi /* host */,
                   int64_t* clusters_a /* host */, int64_t* clusters_b /* host */, void* workspace,
                   size_t ws_bytes, kdb_stream_t stream);

/* Per-phase device times (ms) and counters of the most recent kdb_mst call on
 * this thread: out[0] = rounds, out[1] = init/sweep ms, out[2] = min-edge ms
 * (offer + tie + exchange), out[3] = hook/jump/relabel ms, out[4] = finalize ms,
 * out[5] = in-edge build ms, out[6] = stall (sweep) rounds, out[7] = graph entries
 * read by the per-vertex offer kernel (all rounds), out[8] = filter (inexact: cut)
 * ms, out[9] = heavy-phase ms, out[10] = survivors (inexact: cut entries),
 * out[11] = heavy rounds, out[12] = light threshold (-1: none), out[13] =
 * components after the rows phase, out[14] = overflow fallback, out[15] = filter
 * exceptions, out[16] = filter slow entries, out[17] / out[18] = bytes per rank
 * carried by the MIN all-reduces over component arrays in the rows / heavy
 * phase (counted with or without a communicator; with kdb_mst_inexact the
 * local phase needs none: groups never share a component).  Local-first
 * contraction (multi-rank exact mode): out[19] = 1 when it ran, out[20] / out[21]
 * = max / sum over (virtual) ranks of the local-phase ms, out[22] = transition ms,
 * out[23] = global-phase ms, out[24] = components entering the global phase,
 * out[25] = rows parked for it (all ranks), out[26] = bytes per rank of the
 * transition's all-gathers, out[27] = local rounds (max over ranks), out[28] =
 * global-phase ms of the per-rank offers and ties (all ranks), out[29] = rows
 * phases that reused a kept light ELL (KDB_GRAPH_REUSE).  Returns
 * entries written (at most 32). */
int kdb_last_mst_stats(double* out, int cap);

/* Measurement hooks (bench.py).  kdb_launch_count(): kernels this library has
 * launched so far (library-internal CUB scans/sorts are not counted).  With
 * profiling enabled every kernel launch is bracketed by CUDA events on its
 * stream; kdb_profile_read() returns, per kernel name, the summed device time
 * (ms) and the launch count, names '\n'-separated in `names` (host buffers).
 * Profiling makes kdb_core_mark / kdb_label synchronise their stream. */
void kdb_profile_enable(int on);
void kdb_profile_reset(void);
long long kdb_launch_count(void);
int kdb_profile_read(char* names, size_t names_len, double* ms, long long* counts, int cap);

const char* kdb_status_string(kdb_status s);
const char* kdb_last_error(void);

/* Tuning options: the experiment switches of DESIGN.md §16 (e.g. "KDB_LIGHT":
 * light-phase column count, "KDB_FILTER": 0 disables the heavy filter,
 * "KDB_TRACE": per-round log on stderr).  Every option has a built-in default
 * (the measured configuration); none changes the result, only the way it is
 * computed (the parity suite runs the non-default settings).  The library
 * never reads them from the environment: the caller sets them here (the
 * Python binding's set_option / options(); bench.py forwards KDB_* variables
 * of its own environment once at start).  Process-wide, guarded by a mutex;
 * a call already running may or may not see a change.
 *   kdb_set_option: KDB_EINVAL for an unknown name (nothing changed).
 *   kdb_get_option: 1 and *value (host) if set, 0 if the default applies,
 *                   -1 for an unknown name.
 *   kdb_reset_options: every option back to its default.
 *   kdb_option_name: the i-th known name (host out, static storage); 0 past
 *                    the end. */
kdb_status kdb_set_option(const char* name, long long value);
int kdb_get_option(const char* name, long long* value);
void kdb_reset_options(void);
int kdb_option_name(int i, const char** name);

#ifdef __cplusplus
}
#endif
#endif /* KDB_H_ */
