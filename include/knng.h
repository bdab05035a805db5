/* knng.h -- C-ABI of the exact k-NN graph builders.
 *
 * The clustering stage takes a k-NN graph as input (include/kdb.h); building it
 * is the paper's dominant cost ("constructing k-NNG is the dominant
 * cost"; Table 2: GOFMM on 1,792-7,168 cores, 99% accurate).
 * These builders are EXACT, one GPU each:
 *   - knng_grid  : uniform-grid cell search, 1 <= D <= 5;
 *   - knng_brute : certified brute force, 1 <= D <= 64 (fp32 candidate heaps of
 *                  Kp >= k entries, fp64 re-rank; rows whose certificate fails
 *                  are listed for knng_exact_row).
 * Output convention (the graph convention of kdb.h): row q lists q's k nearest
 * OTHER points, ordered by (fp64 distance, index) where the distance is
 * sqrt(sum_t (x_t - y_t)^2) over fp32 coordinates in dimension order without
 * fused multiply-add; nbr int32 [n][k] ids, dist fp32 [n][k].
 *
 * Conventions: X is a device float32 [n][D] row-major array; every array is a
 * DEVICE pointer owned by the caller unless marked host; work is ordered on
 * `st` (a cudaStream_t); the calls that read results back synchronise it.
 * Return codes: 0 ok, 1 CUDA error, 2 grid overflow (h too small for the
 * bounding box), 3 fallback capacity exceeded, 4 bad arguments (nothing
 * launched).
 */
#ifndef KNNG_H_
#define KNNG_H_

#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Device workspace bytes knng_grid needs for n points. */
size_t knng_grid_ws(int64_t n);

/* Radius estimate for choosing the grid cell size h: for each of the S sample
 * ids samples[s] (device int32[S]), a log2-ladder histogram (64 buckets,
 * bucket j = distances in [r_lo 2^(j/4), r_lo 2^((j+1)/4))) of its distances to
 * all n points -> hist (device uint32 [S][64], zeroed by the call). */
int knng_ladder(const float* X, int64_t n, int D, const int32_t* samples, int S, float r_lo, unsigned int* hist,
                cudaStream_t st);

/* Exact kNN graph by grid cell search.  h > 0: cell edge; lo (host double[D]):
 * the grid origin (<= every coordinate - 2h); span_cells (host): the bounding
 * box extent in cells; diag (host): its diagonal (distance bound for the ring
 * fallback).  nbr/dist: [n][k] outputs.  ws: >= knng_grid_ws(n) bytes.
 * n_fallback (host out): queries that needed rings beyond the 3^D block.
 * 1 <= k <= n-1.  Synchronises st. */
int knng_grid(const float* X, int64_t n, int D, int k, double h, const double* lo, double span_cells, double diag,
              int32_t* nbr, float* dist, void* ws, size_t ws_bytes, cudaStream_t st, int64_t* n_fallback);

/* The same for the query rows [q_begin, q_begin + q_count) only (one rank's
 * contiguous rows of a distributed graph): the grid is built over
 * all n points (every point is a candidate), nbr/dist are [q_count][k] with
 * row r holding query q_begin + r.  Cells holding no such query are skipped.
 * 4 also for a range outside [0, n).  knng_grid == knng_grid_rows(0, n). */
int knng_grid_rows(const float* X, int64_t n, int D, int k, double h, const double* lo, double span_cells,
                   double diag, int64_t q_begin, int64_t q_count, int32_t* nbr, float* dist, void* ws,
                   size_t ws_bytes, cudaStream_t st, int64_t* n_fallback);

/* Certified brute force: per query an fp32 heap of the Kp nearest candidates
 * (k <= Kp <= 256; hs float[n*Kp], hi int32[n*Kp], hcount int32[n] scratch),
 * then an fp64 re-rank into nbr/dist [n][k].  A row whose k-th fp64 distance is
 * not certified below the heap's fp32 bound (with its rounding margin) is
 * written to fail_rows (int32[n]) and counted in n_fail (uint32[1], zeroed by
 * the caller); such rows must be recomputed with knng_exact_row. */
int knng_brute(const float* X, int64_t n, int D, int k, int Kp, float* hs, int32_t* hi, int32_t* hcount,
               int32_t* nbr, float* dist, int32_t* fail_rows, unsigned int* n_fail, cudaStream_t st);

/* fp64 distances of query q to all n points -> out (device double[n]). */
int knng_exact_row(const float* X, int64_t n, int D, int64_t q, double* out, cudaStream_t st);

#ifdef __cplusplus
}
#endif
#endif /* KNNG_H_ */
