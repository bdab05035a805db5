"""epsilon-monotonicity and epsilon-saturation (SURVEY.md §4 layer 5), on the
oracle (-m "not gpu") and on the CUDA path (-m gpu).

For a fixed kNN graph and M (Thm. 2):
  * monotone: eps1 < eps2  =>  core(eps1) is a subset of core(eps2), and every
    core cluster at eps1 lies inside one core cluster at eps2 (the candidate
    edge set only grows with eps, so components only merge);
  * lower saturation: eps < min_i D[i][M-1]  =>  no core point, every label -1,
    empty forest;
  * upper saturation: eps >= max D (rows full)  =>  every point core, and the
    clusters are the connected components of the undirected kNN graph (BFS,
    test-side), the forest has N - #components edges and its weight is Prim's.
Checked with test-side code only (BFS, Prim); nothing here re-types the oracle.
"""
from __future__ import annotations

import heapq

import numpy as np
import pytest

import oracle
from datagen import knn_bruteforce, random_graph


def _points(seed, n=400, d=2):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-3, 3, size=(5, d))
    X = c[rng.integers(0, 5, n)] + 0.3 * rng.standard_normal((n, d))
    return X.astype(np.float32)


def _graphs():
    out = []
    for seed in (0, 1):
        X = _points(seed)
        nbr, dist = knn_bruteforce(X, 12)
        out.append((f"points{seed}", nbr, dist, True))
    nbr, dist = random_graph(300, 10, seed=7, levels=6)
    out.append(("random-ties", nbr, dist, False))
    return out


def _bfs_components(nbr, n):
    adj = [[] for _ in range(n)]
    for i in range(n):
        for J in nbr[i]:
            if J >= 0 and J != i:
                adj[i].append(int(J)); adj[int(J)].append(i)
    lab = np.full(n, -1, np.int64)
    for s in range(n):
        if lab[s] >= 0:
            continue
        lab[s] = s
        st = [s]
        while st:
            u = st.pop()
            for v in adj[u]:
                if lab[v] < 0:
                    lab[v] = s; st.append(v)
    return lab  # = minimum id of the component (s visited in increasing order)


def _prim_weight(nbr, dist, n):
    adj = [[] for _ in range(n)]
    for i in range(n):
        for J, w in zip(nbr[i], dist[i]):
            if J >= 0 and J != i:
                adj[i].append((float(w), int(J))); adj[int(J)].append((float(w), i))
    seen = np.zeros(n, bool)
    tot = 0.0
    for s in range(n):
        if seen[s]:
            continue
        seen[s] = True
        h = list(adj[s]); heapq.heapify(h)
        while h:
            w, v = heapq.heappop(h)
            if seen[v]:
                continue
            seen[v] = True
            tot += w
            for e in adj[v]:
                if not seen[e[1]]:
                    heapq.heappush(h, e)
    return tot


def _eps_ladder(dist, M):
    col = np.sort(dist[:, M - 1].astype(np.float64))
    qs = [col[int(f * (len(col) - 1))] for f in (0.05, 0.3, 0.5, 0.7, 0.95)]
    return [np.float32(q) for q in qs]


def check_monotone(res_list, n):
    """res_list: results in increasing eps order (core: 0/1, labels)."""
    for lo, hi in zip(res_list, res_list[1:]):
        c1, c2 = lo["core"].astype(bool), hi["core"].astype(bool)
        assert not np.any(c1 & ~c2), "core(eps1) must be a subset of core(eps2)"
        l1, l2 = lo["labels"], hi["labels"]
        for lab in np.unique(l1[c1]):
            members = np.flatnonzero(c1 & (l1 == lab))
            assert len(np.unique(l2[members])) == 1, "a cluster at eps1 split at eps2"


def check_saturation(nbr, dist, M, run):
    n = nbr.shape[0]
    lo = np.float32(np.nextafter(np.float32(dist[:, M - 1].min()), np.float32(0)))
    r = run(lo)
    assert r["core"].sum() == 0 and np.all(r["labels"] == -1) and len(r["msf_a"]) == 0
    hi = np.float32(dist[np.isfinite(dist)].max())
    r = run(hi)
    assert r["core"].sum() == n  # rows are full (caller checks), so D[i][M-1] <= max D
    comp = _bfs_components(nbr, n)
    assert np.array_equal(r["labels"], comp.astype(r["labels"].dtype))
    ncomp = len(np.unique(comp))
    assert len(r["msf_a"]) == n - ncomp
    pw = _prim_weight(nbr, dist, n)
    assert abs(r["msf_weight"] - pw) <= 1e-9 * max(pw, 1.0)


def _oracle_run(nbr, dist, M):
    return lambda eps: oracle.kdbscan(nbr, dist, M, np.float32(eps))


@pytest.mark.parametrize("case", range(3))
def test_oracle_eps_monotone_and_saturating(case):
    name, nbr, dist, _ = _graphs()[case]
    M = 5
    run = _oracle_run(nbr, dist, M)
    check_monotone([run(e) for e in _eps_ladder(dist, M)], nbr.shape[0])
    if np.all(nbr >= 0):
        check_saturation(nbr, dist, M, run)


def test_monotone_check_catches_a_split():
    """The checker itself: a labelling where a low-eps cluster is split fails."""
    lo = dict(core=np.array([1, 1, 1]), labels=np.array([0, 0, 0]), msf_a=np.zeros(2))
    hi = dict(core=np.array([1, 1, 1]), labels=np.array([0, 0, 2]), msf_a=np.zeros(1))
    with pytest.raises(AssertionError):
        check_monotone([lo, hi], 3)
    hi2 = dict(core=np.array([1, 0, 1]), labels=np.array([0, -1, 0]), msf_a=np.zeros(1))
    with pytest.raises(AssertionError):
        check_monotone([lo, hi2], 3)


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(3))
@pytest.mark.parametrize("exact", [False, True])
def test_gpu_eps_monotone_and_saturating(case, exact):
    import torch
    import paper_2009_04552_b200 as kdb
    from tests.kdb_harness import result_dict
    name, nbr, dist, is_exact = _graphs()[case]
    if exact and not is_exact:
        pytest.skip("random graph is not an exact kNN graph")
    M = 5
    n = nbr.shape[0]
    g = kdb.Graph(torch.from_numpy(nbr).cuda(), torch.from_numpy(dist).cuda(), n_total=n, exact=exact)

    def run(eps):
        bits, r, lab = kdb.kdbscan(g, M, float(eps))
        torch.cuda.synchronize()
        return result_dict(bits, r, lab, n)

    ladder = _eps_ladder(dist, M)
    res = [run(e) for e in ladder]
    check_monotone(res, n)
    for e, got in zip(ladder, res):  # and each rung equals the oracle
        exp = oracle.kdbscan(nbr, dist, M, e)
        assert np.array_equal(got["labels"], exp["labels"]) and np.array_equal(got["msf_a"], exp["msf_a"])
    # the sweep entry point over the same ladder, descending order, equals the single runs
    sw = kdb.kdbscan_sweep(g, M, [float(e) for e in ladder[::-1]])
    torch.cuda.synchronize()
    for (_, bits, r, lab), got in zip(sw, res[::-1]):
        assert np.array_equal(lab.cpu().numpy(), got["labels"])
    if np.all(nbr >= 0):
        check_saturation(nbr, dist, M, run)
