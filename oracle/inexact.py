"""CPU oracle of the paper's INEXACT MST -- TEST
INFRASTRUCTURE (only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline may use it).

Definition ("Inexact MST"; Alg. 2 + Alg. 4):
vertex-partition I into n groups I_1..I_n (here the contiguous row ranges of
the distributed layout, [floor(pN/n), floor((p+1)N/n))); the
candidate edges of group i split into E_i,local (both endpoints in I_i) and
E_cut (endpoints in different groups).  MST_i,local = the MSF of
(I_i, E_i,local); each local subtree is a super vertex; MST_cut = the MSF of
(super vertices, E_cut); MST_inexact = U_i MST_i,local U MST_cut.  Thm. 3(ii)
(PAPER.md:1082-1086): its clusters are the kNN-DBSCAN clusters; its weight is
not minimal in general.

Ties: every MSF here is taken under the strict edge order O1 of the ORIGINAL
edge (mono(w), min id, max id) (reading #6), also for cut edges between super
vertices, which makes every step's forest unique.

Steps follow the definition literally with Kruskal (sort by O1, union-find)
written out here; the candidate multiset comes from oracle.candidates (pinned).
Pinned in tests/test_inexact.py.
"""
from __future__ import annotations

import numpy as np

import oracle


def _mono(w):
    u = np.asarray(w, np.float32).view(np.uint32).astype(np.int64)
    return np.where(u == 0x80000000, 0, u)


def part_of(ids, N: int, nparts: int):
    """Group of each id under the contiguous split lo_p = floor(p N / n)."""
    ids = np.asarray(ids, np.int64)
    p = (ids * nparts) // max(N, 1)
    lo = lambda q: (q * N) // nparts
    p = np.where(lo(p + 1) <= ids, p + 1, p)
    p = np.where(lo(p) > ids, p - 1, p)
    return p


class _DSU:
    def __init__(self, n):
        self.p = list(range(n))

    def find(self, x):
        while self.p[x] != x:
            self.p[x] = self.p[self.p[x]]
            x = self.p[x]
        return x

    def union(self, a, b):
        a, b = self.find(a), self.find(b)
        if a == b:
            return False
        self.p[max(a, b)] = min(a, b)
        return True


def _kruskal(n, a, b, w, ends):
    """Kruskal over the edges (a, b, w) in O1 order of (w, a, b); `ends` maps an
    edge to the union-find vertices it joins (identity, or super vertices)."""
    order = np.lexsort((b, a, _mono(w)))
    dsu = _DSU(n)
    keep = []
    for e in order.tolist():
        x, y = ends(e)
        if dsu.union(x, y):
            keep.append(e)
    return keep, dsu


def kdbscan_inexact(nbr, dist, M: int, eps, nparts: int, edge_cols=None):
    """Returns dict(core, labels, msf_a, msf_b (sorted by (a, b)), msf_w, msf_weight,
    n_local, n_cut) for the inexact MST over `nparts` contiguous groups."""
    nbr = np.ascontiguousarray(nbr, np.int32)
    dist = np.ascontiguousarray(dist, np.float32)
    n, k = nbr.shape
    core = oracle.core_mark(dist, M, eps)
    a, b, w = oracle.candidates(nbr, dist, core, eps, edge_cols)
    a = a.astype(np.int64); b = b.astype(np.int64)
    pa, pb = part_of(a, n, nparts), part_of(b, n, nparts)
    local = pa == pb
    # step 1: MST_i,local for every group (one Kruskal: local edges never join groups)
    la, lb, lw = a[local], b[local], w[local]
    keep_l, dsu = _kruskal(n, la, lb, lw, lambda e: (int(la[e]), int(lb[e])))
    sup = np.array([dsu.find(v) for v in range(n)], np.int64)  # super vertex of each point
    # step 2: MST_cut over the super vertices, edges still ordered by their own O1 key
    ca, cb, cw = a[~local], b[~local], w[~local]
    keep_c, dsu2 = _kruskal(n, ca, cb, cw, lambda e: (int(sup[ca[e]]), int(sup[cb[e]])))
    fa = np.concatenate([la[keep_l], ca[keep_c]]).astype(np.uint32)
    fb = np.concatenate([lb[keep_l], cb[keep_c]]).astype(np.uint32)
    fw = np.concatenate([lw[keep_l], cw[keep_c]]).astype(np.float32)
    o = np.lexsort((fb, fa))
    fa, fb, fw = fa[o], fb[o], fw[o]
    # labels: canonical minimum core id of the final tree; border rule as the oracle
    root = np.array([dsu2.find(int(sup[v])) for v in range(n)], np.int64)
    cores = np.nonzero(core)[0]
    mn = {}
    for v in cores.tolist():
        r = root[v]
        mn[r] = min(mn.get(r, v), v)
    comp = np.full(n, -1, np.int32)
    for v in cores.tolist():
        comp[v] = mn[root[v]]
    labels = oracle.border(nbr, dist, core, eps, comp)
    # fp64 sum in O1 order of the forest's edges (as oracle_kdbscan)
    ko = np.lexsort((fb, fa, _mono(fw)))
    weight = float(np.sum(fw[ko].astype(np.float64)))
    return dict(core=core, labels=labels, msf_a=fa, msf_b=fb, msf_w=fw, msf_weight=weight,
                n_local=len(keep_l), n_cut=len(keep_c))
