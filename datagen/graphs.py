"""Random kNN-shaped graphs with adversarial structure, and the epsilon rule.

These are inputs only (the ABI accepts ANY valid graph, PAPER.md:517 and
SURVEY.md §8(b)): rows of k (id, weight) entries, weights non-decreasing per
row, self excluded, ``-1``/``+inf`` padding allowed at the row tail.
"""
from __future__ import annotations

import numpy as np


def random_graph(n: int, k: int, seed: int = 0, *, levels: int | None = 16,
                 symmetric: bool = True, pad_frac: float = 0.0,
                 zero_frac: float = 0.0, local: int | None = None):
    """A random directed graph in kNN layout.

    n, k       -- points and row length (k <= n-1)
    levels     -- weights drawn from ``levels`` distinct fp32 values (many ties);
                  None = continuous uniform weights
    symmetric  -- w(i, j) == w(j, i) (a function of the unordered pair); else
                  every entry draws its own weight (asymmetric graph)
    pad_frac   -- fraction of rows whose tail is padded with (-1, +inf)
    zero_frac  -- fraction of pair weights forced to 0.0 (duplicate points)
    local      -- if set, neighbours are drawn from ids within +-local of i
                  (gives long chains / many components); else uniform
    Ties inside a row are stored in RANDOM id order (never assume ascending
    ids among equal weights, SURVEY.md §8(c) reading #18).
    """
    if not (1 <= k <= n - 1):
        raise ValueError("need 1 <= k <= n-1")
    rng = np.random.default_rng(seed)
    nbr = np.empty((n, k), np.int32)
    dist = np.empty((n, k), np.float32)
    salt = rng.integers(1, 2**62)
    lv = None
    if levels is not None:
        lv = np.sort(rng.uniform(0.05, 1.0, size=levels)).astype(np.float32)

    def pair_w(a: np.ndarray, b: np.ndarray) -> np.ndarray:
        lo = np.minimum(a, b).astype(np.uint64)
        hi = np.maximum(a, b).astype(np.uint64)
        h = (lo * np.uint64(0x9E3779B97F4A7C15) ^ (hi + np.uint64(salt))) * np.uint64(0xBF58476D1CE4E5B9)
        h ^= h >> np.uint64(31)
        u = (h >> np.uint64(11)).astype(np.float64) / float(1 << 53)
        if lv is not None:
            w = lv[np.minimum((u * len(lv)).astype(np.int64), len(lv) - 1)]
        else:
            w = (0.05 + 0.95 * u).astype(np.float32)
        z = ((h >> np.uint64(3)) % np.uint64(1000)).astype(np.float64) / 1000.0
        return np.where(z < zero_frac, np.float32(0.0), w).astype(np.float32)

    for i in range(n):
        if local is None:
            cand = rng.choice(n - 1, size=k, replace=False)
            cand = cand + (cand >= i)
        else:
            lo, hi = max(0, i - local), min(n - 1, i + local)
            pool = np.arange(lo, hi + 1)
            pool = pool[pool != i]
            if len(pool) < k:
                extra = np.setdiff1d(np.arange(n), np.append(pool, i))
                pool = np.concatenate([pool, rng.choice(extra, size=k - len(pool), replace=False)])
            cand = rng.choice(pool, size=k, replace=False)
        if symmetric:
            w = pair_w(np.full(k, i), cand)
        else:
            if lv is not None:
                w = lv[rng.integers(0, len(lv), size=k)]
            else:
                w = rng.uniform(0.05, 1.0, size=k).astype(np.float32)
            w = np.where(rng.uniform(size=k) < zero_frac, np.float32(0.0), w).astype(np.float32)
        perm = rng.permutation(k)                 # random order among ties
        cand, w = cand[perm], w[perm]
        o = np.argsort(w, kind="stable")
        nbr[i] = cand[o]
        dist[i] = w[o]
        if pad_frac > 0 and rng.uniform() < pad_frac:
            p = int(rng.integers(1, k + 1))
            nbr[i, k - p:] = -1
            dist[i, k - p:] = np.inf
    return nbr, dist


def eps_from_graph(dist: np.ndarray, M: int, factor: float) -> np.float32:
    """eps = fp32(factor * median_fp64(D[:, M-1])) (SURVEY.md §8(c) reading #21;
    numpy median = mean of the two middle values for even N)."""
    col = np.asarray(dist[:, M - 1], np.float64)
    return np.float32(factor * float(np.median(col)))
