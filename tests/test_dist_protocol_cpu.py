"""The multi-rank EXCHANGE SEQUENCE of DESIGN.md section 7, executed for real on CPU
with torch.distributed 'gloo' at world size 2 and 3 (-m "not gpu").

libkdb.so needs a GPU, so its own collectives cannot run here.  What can be
checked without one is the protocol the library implements: that ranks which
hold ONLY their contiguous rows of the kNN graph, and exchange ONLY what
section 7 lists, arrive at the oracle's result --

  1. core bits: local marking, all-reduce SUM of disjoint bit words (= OR);
  2. local-first phase (optional): Boruvka on the rank's own rows, no exchange;
     a component hooks only along a minimum that is certified from its own rows
     (strictly below the smallest k-th-neighbour distance of its members, the
     exact-graph certificate) and whose far endpoint is local; otherwise it
     freezes (PAPER.md:538-541, 698-751 give the local MST + cut-edge Boruvka;
     this is its exact form);
  3. transition: all-gather of every rank's component ids of its rows;
  4. global phase: per round one all-reduce MIN of the packed keys
     (mono(w), a, b) per component (north_star: "each Boruvka round all-reduces
     (MIN) the packed component keys"), then hook / symmetry break / pointer
     jumping replicated on every rank;
  5. labels: minimum core id per component; border rows on their owner;
  6. output: rank r keeps the forest edges whose smaller endpoint is in its rows.

This numpy model is test code (it is not a product path and is never imported by
the package); it is compared with oracle/ on every rank: core flags, labels,
the MSF edge set, the MSF weight, and the distributed-output contract.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_04552_b200.dist import rank_rows

INF = np.iinfo(np.int64).max


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mono(w):
    u = np.ascontiguousarray(w, np.float32).view(np.uint32).astype(np.int64)
    u[u == 0x80000000] = 0
    return u


def _allreduce(a, op):
    t = torch.from_numpy(np.ascontiguousarray(a))
    dist.all_reduce(t, op=op)
    return t.numpy()


def _jump(parent):
    while True:
        nxt = parent[parent]
        if np.array_equal(nxt, parent):
            return parent
        parent = nxt


def _hook(part, comp_of_vertex, n):
    """Replicated hook of one round: part[c] = the minimum key of component c (INF:
    none).  Returns (new parent over component ids, the chosen keys)."""
    roots = np.nonzero(part < INF)[0]
    ck = part[roots]
    a, b = (ck >> 16) & 0xFFFF, ck & 0xFFFF
    ca, cb = comp_of_vertex[a], comp_of_vertex[b]
    other = np.where(ca == roots, cb, ca)
    parent = np.arange(n, dtype=np.int64)
    parent[roots] = other
    mutual = parent[other] == roots  # both chose the same edge: the smaller id stays a root
    stay = roots[mutual & (roots < other)]
    parent[stay] = stay
    return _jump(parent), np.unique(ck)


def protocol(rank, world, nbr, dst, rb, N, M, eps, local_first):
    """One rank's run; nbr/dst are this rank's rows only (global neighbour ids)."""
    n_loc, k = nbr.shape
    re_ = rb + n_loc
    assert N <= 65536
    # 1. core bits
    words = np.zeros((N + 31) // 32, np.int64)
    for v in np.nonzero(dst[:, M - 1] <= eps)[0] + rb:
        words[v >> 5] |= 1 << (v & 31)
    words = _allreduce(words, dist.ReduceOp.SUM)
    core = ((words[np.arange(N) >> 5] >> (np.arange(N) & 31)) & 1).astype(bool)
    # candidate entries of this rank's rows
    ii, cc = np.nonzero((nbr >= 0) & (dst <= eps))
    i, j = ii + rb, nbr[ii, cc].astype(np.int64)
    keep = core[i] & core[j] & (i != j)
    i, j, w = i[keep], j[keep], dst[ii[keep], cc[keep]]
    key = (_mono(w) << 32) | (np.minimum(i, j) << 16) | np.maximum(i, j)
    comp = np.arange(N, dtype=np.int64)  # entries outside [rb, re_) are unknown until the transition
    chosen = []
    stats = {"local_rounds": 0, "global_rounds": 0, "frozen": 0}
    if local_first:
        # 2. local phase: no exchange.  comp[] is only read at local vertices.
        bound = np.full(N, INF, np.int64)
        bound[rb:re_] = _mono(dst[:, k - 1])  # an unseen in-edge of v weighs >= D[v][k-1] (exact graph)
        frozen = np.zeros(N, bool)
        jloc = (j >= rb) & (j < re_)
        while True:
            ci = comp[i]
            cj = np.where(jloc, comp[np.where(jloc, j, rb)], -1)  # -1: a remote component (kRemote)
            cross = ci != cj
            part = np.full(N, INF, np.int64)
            np.minimum.at(part, ci[cross], key[cross])  # exact mode: the row owner offers to its own component
            has = part < INF
            far = part & 0xFFFF
            near = (part >> 16) & 0xFFFF
            c_ids = np.arange(N)
            # the far endpoint is the one outside the component
            a_in = np.zeros(N, bool)
            a_in[has] = (near[has] >= rb) & (near[has] < re_)
            a_in[has] &= comp[np.where(a_in[has], near[has], rb)] == c_ids[has]
            far_v = np.where(a_in, far, near)
            far_local = (far_v >= rb) & (far_v < re_)
            certified = has & ((part >> 32) < bound) & far_local & ~frozen
            frozen |= has & ~certified
            go = np.where(certified, part, INF)
            if not (go < INF).any():
                break
            parent, ck = _hook(go, comp, N)
            chosen.append(ck)
            # merged components: bound = min over members, frozen = any member frozen
            nb = np.full(N, INF, np.int64)
            np.minimum.at(nb, parent, bound)
            nf = np.zeros(N, bool)
            np.logical_or.at(nf, parent, frozen)
            live = parent == np.arange(N)
            bound, frozen = np.where(live, nb, INF), nf & live
            comp[rb:re_] = parent[comp[rb:re_]]
            stats["local_rounds"] += 1
        stats["frozen"] = int(frozen.sum())
        # 3. transition: every rank's component ids of its rows (ids are global vertex ids of local roots)
        full = np.zeros(N, np.int64)
        full[rb:re_] = comp[rb:re_]
        comp = _allreduce(full, dist.ReduceOp.SUM)
    # 4. global phase: MIN all-reduce of the packed keys per round, offers to both endpoints' components
    while True:
        ci, cj = comp[i], comp[j]
        cross = ci != cj
        part = np.full(N, INF, np.int64)
        np.minimum.at(part, ci[cross], key[cross])
        np.minimum.at(part, cj[cross], key[cross])
        part = _allreduce(part, dist.ReduceOp.MIN)
        if not (part < INF).any():
            break
        parent, ck = _hook(part, comp, N)
        # only the rank that holds a copy of the edge knows its weight: it reports the edge
        chosen.append(ck)
        comp = parent[comp]
        stats["global_rounds"] += 1
    # 5. labels
    cmin = np.full(N, INF, np.int64)
    cv = np.nonzero(core)[0]
    np.minimum.at(cmin, comp[cv], cv)
    lab = np.zeros(N, np.int64)
    for v in range(rb, re_):
        if core[v]:
            lab[v] = cmin[comp[v]]
        else:
            lab[v] = -1
            for c in range(k):
                J = nbr[v - rb, c]
                if J >= 0 and core[J] and dst[v - rb, c] <= eps:
                    lab[v] = cmin[comp[J]]
                    break
    lab = _allreduce(lab, dist.ReduceOp.SUM)
    # 6. output: this rank's a-range of the forest.  Local-phase keys are rank-private; global-phase
    # keys are replicated; either way a rank keeps an edge iff its smaller endpoint is in its rows.
    keys = np.unique(np.concatenate(chosen)) if chosen else np.zeros(0, np.int64)
    a = (keys >> 16) & 0xFFFF
    mine = keys[(a >= rb) & (a < re_)]
    order = np.lexsort((mine & 0xFFFF, (mine >> 16) & 0xFFFF))
    mine = mine[order]
    # the weight travels in the key (mono(w) is the fp32 bit pattern)
    wk = {int(q): float(np.array([q >> 32], np.uint32).view(np.float32)[0]) for q in mine}
    parts = [None] * world
    dist.all_gather_object(parts, [(int((q >> 16) & 0xFFFF), int(q & 0xFFFF), wk[int(q)], int(q)) for q in mine])
    forest = [e for p in parts for e in p]
    return core, lab, forest, stats


def _inputs(case):
    from datagen import knn_bruteforce
    rng = np.random.default_rng(case)
    if case == 0:  # blobs + noise (the C1 recipe, small)
        n, k, M = 1200, 12, 6
        cent = np.stack([np.cos(np.arange(4) * np.pi / 2), np.sin(np.arange(4) * np.pi / 2)], 1)
        X = np.concatenate([cent[t] + 0.05 * rng.standard_normal((275, 2)) for t in range(4)]
                           + [rng.uniform(-1.5, 1.5, (100, 2))]).astype(np.float32)
        X = X[rng.permutation(n)]  # clusters straddle every rank boundary
    elif case == 1:  # duplicates and a lattice: many equal weights (ties), w = 0
        n, k, M = 900, 10, 4
        g = np.stack(np.meshgrid(np.arange(30), np.arange(30)), -1).reshape(-1, 2).astype(np.float32)
        X = g.copy()
        X[rng.integers(0, n, 60)] = X[rng.integers(0, n, 60)]
    else:  # spatially ordered ids (the inertial-order situation: compact rank regions)
        n, k, M = 1500, 16, 8
        X = rng.uniform(0, 1, (n, 3)).astype(np.float32)
        X = X[np.argsort(X[:, 0], kind="stable")]
    nbr, dst = knn_bruteforce(X, k)
    eps = np.float32(np.median(dst[:, M - 1].astype(np.float64)) * 1.5)
    return nbr, dst, M, eps


def _worker(rank, world, port, case, local_first, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        nbr, dst, M, eps = _inputs(case)
        N = len(nbr)
        exp = oracle.kdbscan(nbr, dst, M, eps)
        rb, re_ = rank_rows(N, rank, world)
        mine_n, mine_d = nbr[rb:re_].copy(), dst[rb:re_].copy()
        del nbr, dst  # from here on the rank sees its rows only
        core, lab, forest, stats = protocol(rank, world, mine_n, mine_d, rb, N, M, eps, local_first)
        ok = {
            "core": bool(np.array_equal(core, exp["core"].astype(bool))),
            "labels": bool(np.array_equal(lab, exp["labels"].astype(np.int64))),
            "msf": [(a, b) for a, b, _, _ in forest] == list(zip(exp["msf_a"].tolist(), exp["msf_b"].tolist())),
        }
        wsum = float(np.sum([w for _, _, w, q in sorted(forest, key=lambda e: e[3])]))
        ok["weight"] = abs(wsum - float(exp["msf_weight"])) <= 1e-6 * max(1.0, abs(float(exp["msf_weight"])))
        ok["n_edges"] = len(forest)
        ok.update(stats)
        out[rank] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("local_first", [False, True])
@pytest.mark.parametrize("case", [0, 1, 2])
@pytest.mark.parametrize("world", [2, 3])
def test_exchange_sequence_reaches_the_oracle(world, case, local_first):
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, case, local_first, out), nprocs=world, join=True)
        res = dict(out)
    assert set(res) == set(range(world))
    for r, ok in res.items():
        assert ok["core"] and ok["labels"] and ok["msf"] and ok["weight"], (r, ok)
        assert ok["n_edges"] > 0
    if local_first:
        # the local phase really contracted something, and the global phase had cut work left
        for ok in res.values():
            assert ok["local_rounds"] >= 2 and ok["frozen"] >= 1 and ok["global_rounds"] >= 1, res
