"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/kdb_oracle.cpp) is checked here against things OTHER than
itself: values printed in the paper's worked examples (tests/golden/), classic
DBSCAN by brute force from the points (Thm. 2(i)), Prim's
algorithm (a different MSF algorithm under the same strict order), exhaustive
enumeration of spanning forests on tiny graphs, BFS components, the
cycle-property certificate, Thm. 1 containment and the
brute-force nearest-core border rule (Lemma 1(ii)).  None of the
checkers below calls into oracle/ except through its public entry points.
"""
from __future__ import annotations

import heapq
import itertools
import json
import os
from collections import deque

import numpy as np
import pytest

import oracle
from datagen import knn_bruteforce, random_graph

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- helpers ----
def mono(w) -> int:
    """fp32 bit pattern, -0 -> +0 (SURVEY.md §8(c) reading #6)."""
    u = int(np.float32(w).view(np.uint32))
    return 0 if u == 0x80000000 else u


def key(w, i, j):
    return (mono(w), min(i, j), max(i, j))


def candidate_edges(nbr, dist, core, eps):
    """Independent re-statement of the candidate multiset (test-side code)."""
    n, k = nbr.shape
    E = []
    for i in range(n):
        if not core[i]:
            continue
        for c in range(k):
            J = int(nbr[i, c]); w = dist[i, c]
            if J >= 0 and J != i and core[J] and w <= np.float32(eps):
                E.append((key(w, i, J), np.float32(w)))
    return E


def bfs_components(n, edges, vertices):
    adj = {v: [] for v in vertices}
    for (mw, a, b), _ in edges:
        adj[a].append(b); adj[b].append(a)
    lab = {}
    for s in sorted(vertices):
        if s in lab:
            continue
        lab[s] = s
        dq = deque([s])
        while dq:
            x = dq.popleft()
            for y in adj[x]:
                if y not in lab:
                    lab[y] = s
                    dq.append(y)
    return lab  # s is the minimum id of its component (visited in id order)


def prim_msf(vertices, edges):
    """Prim's algorithm with a heap under the strict key order; returns edge keys."""
    adj = {v: [] for v in vertices}
    for kk, w in edges:
        _, a, b = kk
        adj[a].append((kk, b)); adj[b].append((kk, a))
    seen, out = set(), []
    for s in sorted(vertices):
        if s in seen:
            continue
        seen.add(s)
        h = list(adj[s]); heapq.heapify(h)
        while h:
            kk, y = heapq.heappop(h)
            if y in seen:
                continue
            seen.add(y)
            out.append(kk)
            for e in adj[y]:
                if e[1] not in seen:
                    heapq.heappush(h, e)
    return out


def points_dist64(X):
    X64 = np.asarray(X, np.float32).astype(np.float64)
    n, d = X64.shape
    acc = np.zeros((n, n))
    for t in range(d):
        diff = X64[:, None, t] - X64[None, :, t]
        acc += diff * diff
    return np.sqrt(acc)


def classic_dbscan(X, M, eps):
    """Brute-force DBSCAN from the points (Def. 1-5) with the
    self-excluded count of reading #1 (>= M OTHER points within eps), fp32
    comparison of fp64 distances, border -> nearest core by (fp64 d, index)."""
    D = points_dist64(X)
    F = D.astype(np.float32)
    n = len(X)
    eps = np.float32(eps)
    within = (F <= eps) & ~np.eye(n, dtype=bool)
    core = within.sum(1) >= M
    lab = np.full(n, -1, np.int64)
    for s in range(n):
        if not core[s] or lab[s] >= 0:
            continue
        lab[s] = s
        dq = deque([s])
        while dq:
            x = dq.popleft()
            for y in np.nonzero(within[x] & core)[0]:
                if lab[y] < 0:
                    lab[y] = s
                    dq.append(y)
    out = lab.copy()
    for i in range(n):
        if core[i]:
            continue
        cands = [j for j in np.nonzero(within[i] & core)[0]]
        if cands:
            j = min(cands, key=lambda j: (D[i, j], j))
            out[i] = lab[j]
    return core.astype(np.uint8), out.astype(np.int32)


def clumpy_points(seed, n, d=2, dup_frac=0.1, lattice=False):
    rng = np.random.default_rng(seed)
    if lattice:
        g = int(np.ceil(np.sqrt(n)))
        P = np.array([(i % g, i // g) for i in range(n)], np.float64) * 0.1
    else:
        c = rng.uniform(-1, 1, size=(4, d))
        P = c[rng.integers(0, 4, n)] + 0.15 * rng.standard_normal((n, d))
    nd = int(dup_frac * n)
    if nd:
        P[rng.integers(0, n, nd)] = P[rng.integers(0, n, nd)]
    return P.astype(np.float32)


# --------------------------------------------------------- golden examples ----
def _run_golden(nbr, dist, case):
    r = oracle.kdbscan(np.array(nbr), np.array(dist, np.float32), case["M"], np.float32(case["eps"]))
    assert r["core"].tolist() == case["core"], case["case"]
    msf = sorted(zip(r["msf_a"].tolist(), r["msf_b"].tolist()))
    assert msf == sorted(map(tuple, case["msf"])), case["case"]
    assert r["msf_weight"] == case["msf_weight"], case["case"]
    assert r["labels"].tolist() == case["labels"], case["case"]


def test_golden_w1_fig_cycle():
    g = json.load(open(os.path.join(GOLDEN, "w1_fig_cycle.json")))
    for case in g["cases"]:
        _run_golden(g["nbr"], g["dist"], case)


def test_golden_w2_fig_cut_mst():
    g = json.load(open(os.path.join(GOLDEN, "w2_fig_cut_mst.json")))
    for case in g["cases"]:
        _run_golden(g["nbr"], g["dist"], case)


def test_golden_w3_unit_square_and_duplicate():
    g = json.load(open(os.path.join(GOLDEN, "w3_unit_square.json")))
    # the stored rows are the exact kNN graph of the stored points
    nbr, dist = knn_bruteforce(np.array(g["points"], np.float32), 2)
    assert nbr.tolist() == g["nbr"] and dist.tolist() == g["dist"]
    for case in g["cases"]:
        _run_golden(g["nbr"], g["dist"], case)
    dup = g["dup"]
    nbr, dist = knn_bruteforce(np.array(dup["points"], np.float32), 2)
    assert nbr.tolist() == dup["nbr"] and dist.tolist() == dup["dist"]
    for case in dup["cases"]:
        _run_golden(dup["nbr"], dup["dist"], case)


def test_negative_zero_is_plus_zero():
    """mono(-0) = mono(+0): a -0 copy and a +0 copy of one pair are one key."""
    g = json.load(open(os.path.join(GOLDEN, "w3_unit_square.json")))["dup"]
    dist = np.array(g["dist"], np.float32)
    dist[4, 0] = np.float32(-0.0)   # both copies of {0,4} stored as -0: uncanonicalised
    dist[0, 0] = np.float32(-0.0)   # bits 0x80000000 would sort after w=1 and lose {0,4}
    r = oracle.kdbscan(np.array(g["nbr"]), dist, 2, np.float32(1.0))
    case = g["cases"][0]
    assert sorted(zip(r["msf_a"].tolist(), r["msf_b"].tolist())) == sorted(map(tuple, case["msf"]))
    assert r["labels"].tolist() == case["labels"]


# ------------------------------------------- Thm. 2(i): k = N-1 == DBSCAN ----
@pytest.mark.parametrize("seed,n,M,q", [(0, 60, 1, 0.1), (1, 120, 3, 0.2), (2, 150, 5, 0.15),
                                         (3, 90, 8, 0.3), (4, 200, 4, 0.05), (5, 64, 2, 0.25)])
def test_k_full_equals_classic_dbscan(seed, n, M, q):
    X = clumpy_points(seed, n, lattice=(seed % 3 == 2))
    nbr, dist = knn_bruteforce(X, n - 1)
    eps = np.float32(np.quantile(dist[:, M - 1].astype(np.float64), q + 0.3))
    core_bf, lab_bf = classic_dbscan(X, M, eps)
    r = oracle.kdbscan(nbr, dist, M, eps)
    assert np.array_equal(r["core"], core_bf)
    assert np.array_equal(r["labels"], lab_bf)


# -------------------------------- core flags: closed form from the points ----
@pytest.mark.parametrize("seed", range(4))
def test_core_closed_form(seed):
    X = clumpy_points(seed + 10, 150)
    k, M = 12, 6
    nbr, dist = knn_bruteforce(X, k)
    eps = np.float32(np.median(dist[:, M - 1].astype(np.float64)))
    F = points_dist64(X).astype(np.float32)
    cnt = ((F <= eps) & ~np.eye(len(X), dtype=bool)).sum(1)
    assert np.array_equal(oracle.core_mark(dist, M, eps), (cnt >= M).astype(np.uint8))


# ------------------------------------------- MSF against Prim and BFS --------
@pytest.mark.parametrize("seed,sym,levels,pad,zero", [
    (0, True, 4, 0.0, 0.0), (1, False, 4, 0.1, 0.0), (2, True, None, 0.2, 0.05),
    (3, False, 3, 0.0, 0.1), (4, True, 2, 0.3, 0.0), (5, True, 16, 0.0, 0.2)])
def test_msf_equals_prim_and_components_equal_bfs(seed, sym, levels, pad, zero):
    n, k, M = 300, 6, 2
    nbr, dist = random_graph(n, k, seed, levels=levels, symmetric=sym, pad_frac=pad,
                             zero_frac=zero, local=12 if seed % 2 else None)
    eps = np.float32(np.quantile(dist[np.isfinite(dist)].astype(np.float64), 0.6))
    r = oracle.kdbscan(nbr, dist, M, eps)
    core = (dist[:, M - 1] <= eps)
    E = candidate_edges(nbr, dist, core, eps)
    verts = [v for v in range(n) if core[v]]
    prim = prim_msf(verts, E)
    got = sorted((mono(w), a, b) for a, b, w in zip(r["msf_a"], r["msf_b"], r["msf_w"]))
    assert got == sorted(prim)
    # exact fp64 weight of the forest within the stated tolerance
    wsum = float(np.sum(np.array([np.uint32(m).view(np.float32) for m, _, _ in prim], np.float64)))
    assert abs(r["msf_weight"] - wsum) <= 1e-12 * max(1.0, abs(wsum))
    lab = bfs_components(n, E, verts)
    for v in verts:
        assert r["labels"][v] == lab[v]
    # forest size invariant: |MSF| = #core - #components
    assert len(got) == len(verts) - len(set(lab.values()))


# --------------------------------- exhaustive enumeration on tiny graphs ----
def _enum_msf(vertices, edges):
    """Spanning forest minimising sum(2^rank) over all maximal forests: under a
    strict total order this is the unique MSF (greedy = matroid optimum)."""
    order = sorted(range(len(edges)), key=lambda e: edges[e][0])
    rank = {e: r for r, e in enumerate(order)}
    lab = bfs_components(0, edges, vertices)
    r_size = len(vertices) - len(set(lab.values()))
    best, best_cost = None, None
    for sub in itertools.combinations(range(len(edges)), r_size):
        par = {v: v for v in vertices}

        def f(x):
            while par[x] != x:
                x = par[x]
            return x
        ok = True
        for e in sub:
            _, a, b = edges[e][0]
            ra, rb = f(a), f(b)
            if ra == rb:
                ok = False
                break
            par[ra] = rb
        if not ok:
            continue
        cost = sum(1 << rank[e] for e in sub)
        if best_cost is None or cost < best_cost:
            best, best_cost = sub, cost
    return sorted(edges[e][0] for e in best) if best is not None else []


@pytest.mark.parametrize("seed", range(12))
def test_msf_bruteforce_enumeration_tiny(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(4, 9))
    k = 2 if n < 7 else 1
    nbr, dist = random_graph(n, k, 100 + seed, levels=2 + seed % 3, symmetric=bool(seed % 2))
    eps = np.float32(1.0)
    core = dist[:, 0] <= eps
    E = candidate_edges(nbr, dist, core, eps)
    assert len(E) <= 12
    verts = [v for v in range(n) if core[v]]
    expect = _enum_msf(verts, E)
    r = oracle.kdbscan(nbr, dist, 1, eps)
    got = sorted((mono(w), a, b) for a, b, w in zip(r["msf_a"], r["msf_b"], r["msf_w"]))
    assert got == expect


# -------------------------------------------- cycle-property certificate ----
@pytest.mark.parametrize("seed", range(3))
def test_cycle_property_certificate(seed):
    n, k, M = 400, 8, 3
    nbr, dist = random_graph(n, k, 50 + seed, levels=5, symmetric=bool(seed % 2), local=20)
    eps = np.float32(np.quantile(dist.astype(np.float64), 0.7))
    r = oracle.kdbscan(nbr, dist, M, eps)
    core = dist[:, M - 1] <= eps
    E = candidate_edges(nbr, dist, core, eps)
    tree = [(mono(w), int(a), int(b)) for a, b, w in zip(r["msf_a"], r["msf_b"], r["msf_w"])]
    adj = {v: [] for v in range(n)}
    for kk in tree:
        adj[kk[1]].append((kk[2], kk)); adj[kk[2]].append((kk[1], kk))
    parent, pkey, depth = {}, {}, {}
    for s in range(n):
        if s in parent or not core[s]:
            continue
        parent[s], pkey[s], depth[s] = s, None, 0
        dq = deque([s])
        while dq:
            x = dq.popleft()
            for y, kk in adj[x]:
                if y not in parent:
                    parent[y], pkey[y], depth[y] = x, kk, depth[x] + 1
                    dq.append(y)
    tset = set(tree)

    def path_max(u, v):
        m = None
        while u != v:
            if depth[u] < depth[v]:
                u, v = v, u
            if parent[u] == u:
                return "disconnected"
            m = pkey[u] if m is None else max(m, pkey[u])
            u = parent[u]
        return m

    for kk, _ in E:
        pm = path_max(kk[1], kk[2])
        assert pm != "disconnected", "forest is not spanning"
        if kk not in tset:
            assert pm < kk, "non-tree edge lighter than its tree path"


# ------------------------------- Thm. 1 containment & Lemma 1(ii) border ----
@pytest.mark.parametrize("seed,k,M", [(0, 6, 3), (1, 10, 4), (2, 5, 5), (3, 16, 8)])
def test_thm1_containment_and_border_rule(seed, k, M):
    X = clumpy_points(200 + seed, 180, dup_frac=0.05)
    nbr, dist = knn_bruteforce(X, k)
    eps = np.float32(np.quantile(dist[:, M - 1].astype(np.float64), 0.5))
    r = oracle.kdbscan(nbr, dist, M, eps)
    core_bf, lab_bf = classic_dbscan(X, M, eps)
    assert np.array_equal(r["core"], core_bf)          # Lemma 1(i)
    lab = r["labels"]
    cores = np.nonzero(core_bf)[0]
    # Thm. 1: every kNN-DBSCAN cluster lies inside one DBSCAN cluster
    for c in set(lab[cores].tolist()):
        members = cores[lab[cores] == c]
        assert len(set(lab_bf[members].tolist())) == 1
    assert len(set(lab[cores].tolist())) >= len(set(lab_bf[cores].tolist()))
    # Lemma 1(ii): border set equals DBSCAN's; label = kNN label of the nearest
    # core within eps over ALL points (by (fp64 d, index))
    D = points_dist64(X)
    F = D.astype(np.float32)
    for i in np.nonzero(~core_bf.astype(bool))[0]:
        cand = [j for j in cores if F[i, j] <= eps and j != i]
        if not cand:
            assert lab[i] == -1 and lab_bf[i] == -1
        else:
            j = min(cand, key=lambda j: (D[i, j], j))
            assert lab[i] == lab[j]
    # canonical labels: each label is the minimum core id of its cluster
    for c in set(lab[cores].tolist()):
        assert c == cores[lab[cores] == c].min()


def test_oracle_rejects_bad_arguments():
    nbr = np.zeros((3, 2), np.int32); dist = np.zeros((3, 2), np.float32)
    with pytest.raises(ValueError):
        oracle.kdbscan(nbr, dist, 3, 1.0)      # M > k
    with pytest.raises(ValueError):
        oracle.kdbscan(nbr, dist, 1, 0.0)      # eps not > 0


# ---------------- edge_cols = M: direct M-reachability (Def. 6-9, Thm. 2(ii)) --
def _m_reach_bruteforce(X, M, eps):
    """kNN-DBSCAN clusters of core points straight from Def. 6-9 (PAPER.md:958-
    975) and Lemma 1(i): N_M(p) = the M nearest OTHER points by fp64 distance
    (reading #1), p -M-> q iff p core and (q in N_M(p) or p in N_M(q)); clusters
    = classes of M-reachability over core points (Lemma 3), labelled by their
    minimum id.  Returns (core, N_M sets, label dict)."""
    D = points_dist64(X)
    n = len(X)
    order = np.argsort(D + np.diag(np.full(n, np.inf)), axis=1, kind="stable")
    NM = [set(order[p, :M].tolist()) for p in range(n)]
    F = D.astype(np.float32)
    core = np.array([max(F[p, q] for q in NM[p]) <= np.float32(eps) for p in range(n)])
    edges = []
    for p in range(n):
        for q in range(n):
            if p < q and core[p] and core[q] and (q in NM[p] or p in NM[q]):
                edges.append(((0, p, q), None))
    lab = bfs_components(n, edges, [v for v in range(n) if core[v]])
    return core, NM, lab


@pytest.mark.parametrize("seed,k,M,q", [(0, 12, 3, 0.5), (1, 12, 5, 0.6), (2, 16, 4, 0.7),
                                         (3, 10, 2, 0.8), (4, 20, 6, 0.5), (5, 8, 8, 0.9)])
def test_edge_cols_M_equals_def6_reachability(seed, k, M, q):
    X = clumpy_points(300 + seed, 160, dup_frac=0.0)
    nbr, dist = knn_bruteforce(X, k)
    eps = np.float32(np.quantile(dist[:, M - 1].astype(np.float64), q))
    core_bf, NM, lab = _m_reach_bruteforce(X, M, eps)
    # the graph's first M columns are N_M (continuous points: no distance ties)
    assert all(set(nbr[p, :M].tolist()) == NM[p] for p in range(len(X)))
    r = oracle.kdbscan(nbr, dist, M, eps, edge_cols=M)
    assert np.array_equal(r["core"].astype(bool), core_bf)
    for v, c in lab.items():
        assert r["labels"][v] == c
    # the MSF is Prim's forest of the candidate edges of columns < M
    core = core_bf
    E = candidate_edges(nbr[:, :M].copy(), dist[:, :M].copy(), core, eps)
    got = sorted((mono(w), a, b) for a, b, w in zip(r["msf_a"], r["msf_b"], r["msf_w"]))
    assert got == sorted(prim_msf([v for v in range(len(X)) if core[v]], E))
    # border rule unchanged (Lemma 1(ii) only looks inside N_M(p)): a non-core
    # point takes the label of the first core entry of its row within eps
    for i in np.nonzero(~core)[0]:
        js = [int(nbr[i, c]) for c in range(k) if dist[i, c] <= eps and core[nbr[i, c]]]
        assert r["labels"][i] == (lab[js[0]] if js else -1)


def test_edge_cols_refines_all_k_and_default_is_k():
    """Fewer candidate edges => every edge_cols=M cluster lies inside one
    all-k cluster (the argument of Thm. 1 applied to edge subsets); edge_cols=k
    is the default exactly; and the restriction is not vacuous on this input."""
    finer_somewhere = False
    for seed in range(6):
        X = clumpy_points(400 + seed, 200, dup_frac=0.05)
        k, M = 16, 3
        nbr, dist = knn_bruteforce(X, k)
        eps = np.float32(np.quantile(dist[:, k - 1].astype(np.float64), 0.7))
        rk = oracle.kdbscan(nbr, dist, M, eps)
        rk2 = oracle.kdbscan(nbr, dist, M, eps, edge_cols=k)
        for f in ("core", "labels", "msf_a", "msf_b", "msf_w"):
            assert np.array_equal(rk[f], rk2[f])
        assert rk["msf_weight"] == rk2["msf_weight"]
        rm = oracle.kdbscan(nbr, dist, M, eps, edge_cols=M)
        cores = np.nonzero(rk["core"])[0]
        for c in set(rm["labels"][cores].tolist()):
            assert len(set(rk["labels"][cores[rm["labels"][cores] == c]].tolist())) == 1
        nm, nk = len(set(rm["labels"][cores].tolist())), len(set(rk["labels"][cores].tolist()))
        assert nm >= nk
        finer_somewhere |= nm > nk
    assert finer_somewhere


def test_edge_cols_bad_arguments():
    nbr = np.zeros((3, 2), np.int32); dist = np.zeros((3, 2), np.float32)
    for bad in (0, 3):
        with pytest.raises(ValueError):
            oracle.kdbscan(nbr, dist, 1, 1.0, edge_cols=bad)
