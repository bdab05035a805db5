"""CPU oracle for clustering quality -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
it.  The paper reports NMI ("clustering accuracy (NMI,
higher is better)") without a formula; the convention is SPEC.md:421-428:

    NMI(A, B) = 2 I(A; B) / (H(A) + H(B))     (arithmetic-mean normalisation,
                                               natural log, joint label histogram)
    NOISE (-1) points form ONE shared pseudo-cluster per labelling;
    both entropies 0 -> 1 (identical partitions); I = 0 -> 0;
    exactly one entropy 0 (partitions differ) -> 0.

cluster_count(A) = number of distinct non-NOISE labels.

Written as the definition: the joint histogram by np.unique over label pairs,
then the sums over cells in fp64.  Pinned in tests/test_nmi.py (SPEC's worked
examples, a hand-computed 2x3 table, sklearn's independent implementation,
symmetry and permutation invariance).
"""
from __future__ import annotations

import numpy as np


def nmi(a, b) -> float:
    a = np.asarray(a, np.int64)
    b = np.asarray(b, np.int64)
    if a.shape != b.shape:
        raise ValueError("length mismatch")
    n = a.size
    if n == 0:
        return 1.0
    # joint cells with their marginals, p_ab log(p_ab / (p_a p_b)) summed
    pairs, n_ab = np.unique(np.stack([a, b], 1), axis=0, return_counts=True)
    ua, n_a = np.unique(a, return_counts=True)
    ub, n_b = np.unique(b, return_counts=True)
    p_ab = n_ab / n
    p_a = (n_a / n)[np.searchsorted(ua, pairs[:, 0])]
    p_b = (n_b / n)[np.searchsorted(ub, pairs[:, 1])]
    I = float(np.sum(p_ab * np.log(p_ab / (p_a * p_b))))
    Ha = float(-np.sum((n_a / n) * np.log(n_a / n)))
    Hb = float(-np.sum((n_b / n) * np.log(n_b / n)))
    if Ha == 0.0 and Hb == 0.0:
        return 1.0
    if Ha == 0.0 or Hb == 0.0:
        return 0.0
    return float(2.0 * I / (Ha + Hb))


def cluster_count(a) -> int:
    a = np.asarray(a, np.int64)
    return int(np.unique(a[a != -1]).size)
