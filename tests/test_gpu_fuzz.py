"""Property-based GPU <-> oracle parity (pytest -m gpu): hypothesis draws graph
shapes and parameters -- n, k, M, weight ties (few levels), padding, zero
weights, asymmetry, id locality, eps quantile, exact / general mode, the edge
set (all k / edge_cols), sim ranks, the light threshold -- and every drawn case
must be bit-identical to the oracle.  Derandomised (a fixed example set) so a
CI failure reproduces."""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings, strategies as st

from datagen import knn_bruteforce, random_graph
from tests.kdb_harness import assert_parity, oracle_run, run_gpu

pytestmark = pytest.mark.gpu


@st.composite
def cases(draw):
    n = draw(st.integers(2, 2500))
    k = draw(st.integers(1, min(40, n - 1)))
    M = draw(st.integers(1, k))
    return dict(
        n=n, k=k, M=M, seed=draw(st.integers(0, 2**31 - 1)),
        levels=draw(st.sampled_from([None, 1, 2, 3, 8, 64])),
        symmetric=draw(st.booleans()),
        pad=draw(st.sampled_from([0.0, 0.1, 0.5])),
        zero=draw(st.sampled_from([0.0, 0.05, 0.3])),
        local=draw(st.sampled_from([None, 3, 20, 200])),
        q=draw(st.floats(0.02, 1.0)),
        edge_cols=draw(st.sampled_from([0, M, max(1, k // 2)])),
        P=draw(st.sampled_from([0, 2, 3])),
        light=draw(st.sampled_from(["1", "2", "4", "10"])),
    )


@settings(max_examples=200, deadline=None, derandomize=True, suppress_health_check=list(HealthCheck))
@given(c=cases())
def test_fuzz_random_graphs(c):
    import paper_2009_04552_b200 as kdb
    assert torch.cuda.is_available()
    nbr, dist = random_graph(c["n"], c["k"], c["seed"], levels=c["levels"], symmetric=c["symmetric"],
                             pad_frac=c["pad"], zero_frac=c["zero"], local=c["local"])
    fin = dist[np.isfinite(dist)].astype(np.float64)
    eps = np.float32(np.quantile(fin, c["q"])) if fin.size else np.float32(1.0)
    if not eps > 0:
        eps = np.float32(1e-3)
    kdb.set_option("KDB_LIGHT", c["light"])
    try:
        exp = oracle_run(nbr, dist, c["M"], eps, edge_cols=c["edge_cols"] or None)
        got = run_gpu(nbr, dist, c["M"], eps, exact=False, edge_cols=c["edge_cols"],
                      comm=kdb.Comm.sim(c["P"]) if c["P"] else None)
        assert_parity(got, exp)
    finally:
        kdb.reset_options()


@settings(max_examples=80, deadline=None, derandomize=True, suppress_health_check=list(HealthCheck))
@given(n=st.integers(3, 2000), d=st.integers(1, 4), k=st.integers(1, 24), dup=st.floats(0.0, 0.3),
       f=st.floats(0.3, 4.0), seed=st.integers(0, 2**31 - 1), P=st.sampled_from([0, 2, 4]))
def test_fuzz_exact_point_graphs(n, d, k, dup, f, seed, P):
    """Exact kNN graphs of random point sets (the KDB_GRAPH_EXACT certificate
    path), duplicates included."""
    import paper_2009_04552_b200 as kdb
    k = min(k, n - 1)
    rng = np.random.default_rng(seed)
    X = rng.uniform(size=(n, d)).astype(np.float32)
    nd = int(dup * n)
    if nd:
        X[rng.integers(0, n, nd)] = X[rng.integers(0, n, nd)]
    nbr, dist = knn_bruteforce(X, k)
    M = max(1, k // 2)
    col = dist[:, M - 1].astype(np.float64)
    eps = np.float32(f * float(np.median(col)))
    if not eps > 0:
        eps = np.float32(1e-3)
    exp = oracle_run(nbr, dist, M, eps)
    got = run_gpu(nbr, dist, M, eps, exact=True, comm=kdb.Comm.sim(P) if P else None)
    assert_parity(got, exp)
