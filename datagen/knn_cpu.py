"""Exact k-NN graph by CPU brute force (input construction, not the hot path).

Graph convention (SURVEY.md §8(c) reading #1 and §8(d)):
  * rows EXCLUDE self; ``nbr[i, c]`` is the id of i's (c+1)-th nearest other point;
  * distances are fp64 ``sqrt(sum_t (x_t - y_t)^2)`` from fp32 coordinates
    promoted to fp64, the sum accumulated in dimension order (no fusion);
  * each row is ordered by (fp64 distance, index) and then stored as fp32
    ``dist`` / int32 ``nbr``.
Only for small N (tests, C1); large configs use the GPU builder in
``datagen/csrc/knng.cu`` which computes the same quantities.
"""
from __future__ import annotations

import numpy as np


def _dist_rows(X64: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """fp64 distances from points ``rows`` to every point, dimension-ordered sum."""
    Q = X64[rows]
    acc = np.zeros((len(rows), X64.shape[0]), np.float64)
    for t in range(X64.shape[1]):
        diff = Q[:, t:t + 1] - X64[None, :, t]
        acc += diff * diff
    return np.sqrt(acc)


def knn_rows_bruteforce(X: np.ndarray, rows: np.ndarray, k: int):
    """Exact self-excluded kNN rows for query ids ``rows`` against all of X."""
    X64 = np.asarray(X, np.float32).astype(np.float64)
    rows = np.asarray(rows, np.int64)
    N = X64.shape[0]
    if not (1 <= k <= N - 1):
        raise ValueError("need 1 <= k <= N-1")
    nbr = np.empty((len(rows), k), np.int32)
    dist = np.empty((len(rows), k), np.float32)
    chunk = max(1, min(len(rows), int(2e7 // max(N, 1))))
    for s in range(0, len(rows), chunk):
        r = rows[s:s + chunk]
        D = _dist_rows(X64, r)
        D[np.arange(len(r)), r] = np.inf          # exclude self
        # stable argsort on distance => ties ordered by ascending index
        order = np.argsort(D, axis=1, kind="stable")[:, :k]
        nbr[s:s + len(r)] = order.astype(np.int32)
        dist[s:s + len(r)] = np.take_along_axis(D, order, axis=1).astype(np.float32)
    return nbr, dist


def knn_bruteforce(X: np.ndarray, k: int):
    """Exact self-excluded kNN graph of all points (O(N^2); N up to ~2e4)."""
    return knn_rows_bruteforce(X, np.arange(X.shape[0]), k)
