"""The N>1 path's host logic on CPU with torch.distributed 'gloo', world size 2
(-m "not gpu"): contiguous row ranges, the NCCL unique-id broadcast, the
max-over-ranks step time, and the collective semantics the library relies on
(core bits: SUM of disjoint per-rank bits == OR; per-round keys: MIN of
per-rank partial minima == the single-process minimum), checked against a
single-process computation on the same seeded inputs."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_04552_b200.dist import gather_rows, max_over_ranks, rank_rows, share_nccl_id


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [0, 1, 7, 1000, 64_000_003])
def test_rank_rows_partition(n, world):
    ranges = [rank_rows(n, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        # 1. the 128-byte id created on rank 0 arrives unchanged everywhere
        uid = share_nccl_id(rank, lambda: bytes(range(128)))
        res["uid_ok"] = uid == bytes(range(128))
        # 2. the step time is the slowest rank's
        res["max"] = max_over_ranks(1.0 + rank)
        # 3. core bits: each rank marks its own rows; SUM of disjoint bits == OR
        rng = np.random.default_rng(0)
        N = 1000
        core = rng.uniform(size=N) < 0.6
        rb, re_ = rank_rows(N, rank, world)
        words = np.zeros((N + 31) // 32, np.int64)
        for v in range(rb, re_):
            if core[v]:
                words[v >> 5] |= 1 << (v & 31)
        t = torch.from_numpy(words)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        full = np.zeros_like(words)
        for v in range(N):
            if core[v]:
                full[v >> 5] |= 1 << (v & 31)
        res["bits_ok"] = bool(np.array_equal(t.numpy(), full))
        # 4. per-round keys: MIN of per-rank partial minima == global minimum
        C = 50
        comp = rng.integers(0, C, N)
        key = rng.integers(0, 2**62, N, dtype=np.int64)
        part = np.full(C, np.iinfo(np.int64).max, np.int64)
        np.minimum.at(part, comp[rb:re_], key[rb:re_])
        t = torch.from_numpy(part)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ref = np.full(C, np.iinfo(np.int64).max, np.int64)
        np.minimum.at(ref, comp, key)
        res["min_ok"] = bool(np.array_equal(t.numpy(), ref))
        # 5. the eps rule's column: every rank's rows (uneven counts) gathered in
        #    rank order equal the whole column on every rank (bench.py per-rank build)
        colfull = rng.uniform(size=N + world).astype(np.float32)
        rb2, re2 = rank_rows(N + world, rank, world)
        g = gather_rows(torch.from_numpy(colfull[rb2:re2].copy()))
        res["gather_ok"] = bool(np.array_equal(g.numpy(), colfull))
        # 6. multi-rank MSF output (kdb.h): rank r keeps the edges whose smaller
        #    endpoint lies in its rows, sorted by (a, b); concatenated in rank
        #    order they are the whole sorted forest
        import oracle
        from datagen import knn_bruteforce
        X = np.random.default_rng(5).standard_normal((300, 2)).astype(np.float32)
        nbr, dstt = knn_bruteforce(X, 8)
        ex = oracle.kdbscan(nbr, dstt, 4, np.float32(np.median(dstt[:, 3]) * 1.5))
        a, b = ex["msf_a"].astype(np.int64), ex["msf_b"].astype(np.int64)
        perm = np.random.default_rng(rank).permutation(len(a))  # emission order is arbitrary
        ra, rb_ = rank_rows(300, rank, world)
        keep = perm[(a[perm] >= ra) & (a[perm] < rb_)]
        mine = sorted(zip(a[keep].tolist(), b[keep].tolist()))
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        res["msf_ok"] = [e for p_ in allp for e in p_] == list(zip(a.tolist(), b.tolist()))
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_world2_host_logic(world):
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert set(res) == set(range(world))
    for r in res.values():
        assert r["uid_ok"] and r["bits_ok"] and r["min_ok"] and r["gather_ok"] and r["msf_ok"]
        assert r["max"] == float(world)
