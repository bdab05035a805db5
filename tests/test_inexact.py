"""Pins for the inexact-MST oracle (oracle/inexact.py)
and, with a GPU, parity of kdb_mst_inexact against it."""
from __future__ import annotations

from collections import defaultdict, deque

import numpy as np
import pytest

import oracle
from datagen import eps_from_graph, knn_bruteforce, random_graph
from oracle import inexact as oinx
from tests.test_oracle_pins import candidate_edges, clumpy_points, key, mono, prim_msf


def _cases():
    out = []
    for seed in range(4):
        nbr, dist = random_graph(400, 8, seed, levels=4 if seed % 2 else None, symmetric=bool(seed % 2),
                                 pad_frac=0.1 * (seed % 3), local=20 if seed < 2 else None)
        eps = np.float32(np.quantile(dist[np.isfinite(dist)].astype(np.float64), 0.6))
        out.append((nbr, dist, 3, eps))
    for seed in range(2):
        X = clumpy_points(700 + seed, 300, dup_frac=0.05)
        nbr, dist = knn_bruteforce(X, 12)
        out.append((nbr, dist, 4, eps_from_graph(dist, 4, 1.5)))
    return out


CASES = _cases()


@pytest.mark.parametrize("ci", range(len(CASES)))
@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
def test_thm3_labels_equal_exact_and_forest_invariants(ci, P):
    nbr, dist, M, eps = CASES[ci]
    ex = oracle.kdbscan(nbr, dist, M, eps)
    r = oinx.kdbscan_inexact(nbr, dist, M, eps, P)
    assert np.array_equal(r["core"], ex["core"])
    assert np.array_equal(r["labels"], ex["labels"])            # Thm. 3(ii)
    core = ex["core"].astype(bool)
    n_cl = len(set(ex["labels"][core].tolist()))
    assert len(r["msf_a"]) == int(core.sum()) - n_cl          # a spanning forest of every cluster
    E = candidate_edges(nbr, dist, core, eps)
    cand = {kk for kk, _ in E}
    for a, b, w in zip(r["msf_a"].tolist(), r["msf_b"].tolist(), r["msf_w"]):
        assert key(w, a, b) in cand                            # every forest edge is a candidate edge
    assert r["msf_weight"] >= ex["msf_weight"] - 1e-9 * abs(ex["msf_weight"])  # the exact MSF is minimal
    if P == 1:
        assert np.array_equal(r["msf_a"], ex["msf_a"]) and np.array_equal(r["msf_b"], ex["msf_b"])
        assert r["msf_weight"] == ex["msf_weight"]


def test_inexact_differs_from_exact_somewhere():
    worse = 0
    for nbr, dist, M, eps in CASES:
        ex = oracle.kdbscan(nbr, dist, M, eps)
        r = oinx.kdbscan_inexact(nbr, dist, M, eps, 5)
        worse += r["msf_weight"] > ex["msf_weight"]
    assert worse > 0  # the restriction to local edges does change the forest


@pytest.mark.parametrize("ci", range(len(CASES)))
@pytest.mark.parametrize("P", [2, 3, 5])
def test_local_parts_are_prim_and_cut_part_obeys_cycle_property(ci, P):
    nbr, dist, M, eps = CASES[ci]
    n = nbr.shape[0]
    r = oinx.kdbscan_inexact(nbr, dist, M, eps, P)
    core = r["core"].astype(bool)
    E = candidate_edges(nbr, dist, core, eps)
    part = oinx.part_of(np.arange(n), n, P)
    F = {key(w, a, b) for a, b, w in zip(r["msf_a"].tolist(), r["msf_b"].tolist(), r["msf_w"])}
    # local: per group, the forest's internal edges are Prim's MSF of the group's local edges
    for p in range(P):
        El = [(kk, w) for kk, w in E if part[kk[1]] == p and part[kk[2]] == p]
        verts = [v for v in range(n) if core[v] and part[v] == p]
        prim = set(prim_msf(verts, El))
        assert {kk for kk in F if part[kk[1]] == p and part[kk[2]] == p} == prim
    # super vertices: components of the local forest
    adj = defaultdict(list)
    for kk in F:
        if part[kk[1]] == part[kk[2]]:
            adj[kk[1]].append(kk[2]); adj[kk[2]].append(kk[1])
    sup = {}
    for s in range(n):
        if not core[s] or s in sup:
            continue
        sup[s] = s
        dq = deque([s])
        while dq:
            x = dq.popleft()
            for y in adj[x]:
                if y not in sup:
                    sup[y] = s
                    dq.append(y)
    # cut forest on super vertices; every other cut edge closes a cycle of smaller keys
    cadj = defaultdict(list)
    for kk in F:
        if part[kk[1]] != part[kk[2]]:
            x, y = sup[kk[1]], sup[kk[2]]
            assert x != y
            cadj[x].append((y, kk)); cadj[y].append((x, kk))

    def path_max(s, t):
        best = {s: None}
        dq = deque([s])
        while dq:
            x = dq.popleft()
            for y, kk in cadj[x]:
                if y not in best:
                    best[y] = kk if best[x] is None else max(best[x], kk)
                    dq.append(y)
        return best.get(t, "none")

    for kk, _ in E:
        if part[kk[1]] == part[kk[2]] or kk in F:
            continue
        x, y = sup[kk[1]], sup[kk[2]]
        if x == y:
            continue
        pm = path_max(x, y)
        assert pm != "none" and pm < kk


def test_part_of_matches_ranges():
    for N, P in [(10, 3), (7, 7), (1000, 8), (5, 1)]:
        lo = [(p * N) // P for p in range(P + 1)]
        exp = np.concatenate([np.full(lo[p + 1] - lo[p], p) for p in range(P)])
        assert np.array_equal(oinx.part_of(np.arange(N), N, P), exp)


# ------------------------------------------------------------- GPU parity ----
def _gpu_inexact(nbr, dist, M, eps, P, edge_cols=0):
    import torch
    import paper_2009_04552_b200 as kdb
    g = kdb.Graph(torch.from_numpy(nbr).cuda(), torch.from_numpy(dist).cuda(), n_total=nbr.shape[0],
                  edge_cols=edge_cols)
    bits = kdb.core_mark(g, M, float(eps))
    r = kdb.mst_inexact(g, float(eps), bits, P)
    lab = kdb.label(g, float(eps), bits, r.comp)
    torch.cuda.synchronize()
    return dict(core=kdb.unpack_core(bits, nbr.shape[0]).numpy(), comp=r.comp.cpu().numpy(),
                labels=lab.cpu().numpy(), msf_a=r.a.cpu().numpy().astype(np.uint32),
                msf_b=r.b.cpu().numpy().astype(np.uint32), msf_w=r.w.cpu().numpy(), msf_weight=r.weight,
                stats=r.stats)


@pytest.mark.gpu
@pytest.mark.parametrize("ci", range(len(CASES)))
@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
def test_kdb_mst_inexact_parity(ci, P):
    from tests.kdb_harness import assert_parity
    nbr, dist, M, eps = CASES[ci]
    exp = oinx.kdbscan_inexact(nbr, dist, M, eps, P)
    assert_parity(_gpu_inexact(nbr, dist, M, eps, P), exp)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4, 7])
def test_kdb_mst_inexact_c1(P):
    from datagen import gen_c1
    from tests.kdb_harness import assert_parity
    X, _ = gen_c1(0)
    nbr, dist = knn_bruteforce(X, 16)
    for f, ec in ((1.5, 0), (1.0, 0), (1.5, 8)):
        eps = eps_from_graph(dist, 8, f)
        exp = oinx.kdbscan_inexact(nbr, dist, 8, eps, P, edge_cols=ec or None)
        got = _gpu_inexact(nbr, dist, 8, eps, P, edge_cols=ec)
        assert_parity(got, exp)
        ex = oracle.kdbscan(nbr, dist, 8, eps, edge_cols=ec or None)
        assert np.array_equal(got["labels"], ex["labels"])   # Thm. 3(ii)
        assert got["msf_weight"] >= ex["msf_weight"] * (1 - 1e-12)
