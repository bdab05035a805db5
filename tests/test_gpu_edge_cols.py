"""GPU <-> oracle parity for the paper's own edge set and the multi-eps sweep
(pytest -m gpu).

edge_cols = M: candidate edges only from the first M columns of each row --
direct M-reachability, Def. 6, Alg. 2's bound L[i] <= M
(PAPER.md:566); Thm. 2(ii).  The oracle side is
oracle.kdbscan(..., edge_cols=M), pinned in tests/test_oracle_pins.py against
brute-force Def. 6-9 clusters.  The sweep reuses one resident graph and one
workspace for every eps (Fig. eps_mnist protocol).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from datagen import eps_from_graph, gen_c1, knn_bruteforce, random_graph
from tests.kdb_harness import assert_parity, oracle_run, result_dict, run_gpu
from tests.kdb_harness import kdb_opt as _kdb_opt
from tests.test_gpu_parity import RANDOM_CASES

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2009_04552_b200 as kdb
    kdb.lib()


@pytest.fixture(scope="module")
def c1_graph():
    X, _ = gen_c1(0)
    nbr, dist = knn_bruteforce(X, 16)
    return nbr, dist


def _eps(dist, q):
    return np.float32(np.quantile(dist[np.isfinite(dist)].astype(np.float64), q))


@pytest.mark.parametrize("which", ["1", "M", "k-1", "k"])
@pytest.mark.parametrize("case", RANDOM_CASES)
def test_random_graphs_edge_cols(case, which):
    n, k, M, seed, levels, sym, pad, zero, local, q = case
    nbr, dist = random_graph(n, k, seed, levels=levels, symmetric=sym, pad_frac=pad, zero_frac=zero, local=local)
    kc = {"1": 1, "M": M, "k-1": max(k - 1, 1), "k": k}[which]
    eps = _eps(dist, q)
    exp = oracle_run(nbr, dist, M, eps, edge_cols=kc)
    assert_parity(run_gpu(nbr, dist, M, eps, edge_cols=kc), exp)


@pytest.mark.parametrize("light", ["2", "4", "10"])
@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("P", [0, 3])
def test_c1_edge_cols_M(c1_graph, light, exact, P, monkeypatch):
    """C1 at full size with the Def. 6 edge set; filtered (light < M) and
    unfiltered (light >= M) paths, exact-graph certificate on and off, sim ranks."""
    import paper_2009_04552_b200 as kdb
    _kdb_opt("KDB_LIGHT", light)
    nbr, dist = c1_graph
    eps = eps_from_graph(dist, 8, 1.5)
    exp = oracle_run(nbr, dist, 8, eps, edge_cols=8)
    got = run_gpu(nbr, dist, 8, eps, exact=exact, edge_cols=8, comm=kdb.Comm.sim(P) if P else None)
    assert_parity(got, exp)
    # the restriction matters on C1: finer clustering than all-k (Thm. 1 argument)
    allk = oracle_run(nbr, dist, 8, eps)
    core = exp["core"].astype(bool)
    assert len(np.unique(exp["labels"][core])) >= len(np.unique(allk["labels"][core]))
    assert len(exp["msf_a"]) <= len(allk["msf_a"])


def test_points_exact_graphs_edge_cols():
    """Exact kNN graphs of point sets with duplicates: the certificate must
    stay valid on the truncated (edge_cols-NN) graph."""
    rng = np.random.default_rng(11)
    for n, d, k, M in [(3000, 2, 12, 4), (2500, 3, 20, 10), (2000, 2, 8, 8)]:
        X = rng.uniform(0, 1, size=(n, d)).astype(np.float32)
        X[rng.integers(0, n, n // 20)] = X[rng.integers(0, n, n // 20)]
        nbr, dist = knn_bruteforce(X, k)
        for f in (1.0, 2.0):
            eps = eps_from_graph(dist, M, f)
            exp = oracle_run(nbr, dist, M, eps, edge_cols=M)
            assert_parity(run_gpu(nbr, dist, M, eps, exact=True, edge_cols=M), exp)


@pytest.mark.parametrize("edge_cols", [None, 8])
def test_c1_multi_eps_sweep(c1_graph, edge_cols):
    """kdbscan_sweep: one resident graph, one workspace, many eps; every eps
    equals an independent oracle run (ascending and descending order)."""
    import paper_2009_04552_b200 as kdb
    nbr, dist = c1_graph
    g = kdb.Graph(torch.from_numpy(nbr).cuda(), torch.from_numpy(dist).cuda(), n_total=nbr.shape[0], exact=True)
    factors = [0.3, 0.6, 1.0, 1.5, 2.5, 10.0]
    eps_list = [eps_from_graph(dist, 8, f) for f in factors]
    for order in (eps_list, eps_list[::-1]):
        res = kdb.kdbscan_sweep(g, 8, order, edge_cols=edge_cols)
        torch.cuda.synchronize()
        for eps, bits, r, lab in res:
            got = result_dict(bits, r, lab, nbr.shape[0])
            assert_parity(got, oracle_run(nbr, dist, 8, np.float32(eps), edge_cols=edge_cols))


def test_edge_cols_default_equals_k(c1_graph):
    nbr, dist = c1_graph
    eps = eps_from_graph(dist, 8, 1.5)
    a = run_gpu(nbr, dist, 8, eps, exact=True)
    b = run_gpu(nbr, dist, 8, eps, exact=True, edge_cols=16)
    for key in ("core", "comp", "labels", "msf_a", "msf_b", "msf_w"):
        assert np.array_equal(a[key], b[key])
    assert a["msf_weight"] == b["msf_weight"]
