"""eps sweep with the light ELL kept across calls (KDB_GRAPH_REUSE; Fig.
eps_mnist protocol: one kNN graph, many eps), against the
oracle at every eps (pytest -m gpu).  The ELL and the per-row certificate
bounds depend on the graph and the light threshold (a fixed column's median),
not on eps, so every call after the first reuses them; the results must be the
oracle's whatever the order of the eps values, and a reuse request the library
cannot honour (another graph, another edge_cols) must fall back to a rebuild."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2009_04552_b200 as kdb
from datagen import eps_from_graph, gen_c1, knn_bruteforce
from tests.kdb_harness import assert_parity, oracle_run, result_dict
from tests.kdb_harness import kdb_opt as _kdb_opt

pytestmark = pytest.mark.gpu


def _points(seed, n, d, k):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-3, 3, size=(5, d))
    X = (c[rng.integers(0, 5, n)] + 0.4 * rng.standard_normal((n, d))).astype(np.float32)
    X[rng.integers(0, n, n // 30)] = X[rng.integers(0, n, n // 30)]  # duplicates: w = 0 ties
    return knn_bruteforce(X, k)


@pytest.mark.parametrize("case", ["c1_light10", "k48"])
@pytest.mark.parametrize("order", ["up", "down"])
def test_sweep_reuses_the_ell(case, order, monkeypatch):
    if case == "c1_light10":
        X, _ = gen_c1(0)
        nbr, dist = knn_bruteforce(X, 16)
        M = 8
        _kdb_opt("KDB_LIGHT", "10")  # k = 16: the light/heavy split only when asked for
    else:
        nbr, dist = _points(3, 3000, 3, 48)
        M = 12
    factors = [0.6, 0.9, 1.2, 1.6, 2.5]
    if order == "down":
        factors = factors[::-1]
    g = kdb.Graph(torch.from_numpy(nbr).cuda(), torch.from_numpy(dist).cuda(), n_total=len(nbr), exact=True)
    out = kdb.kdbscan_sweep(g, M, [float(eps_from_graph(dist, M, f)) for f in factors])
    torch.cuda.synchronize()
    reused = 0
    for i, (eps, bits, r, lab) in enumerate(out):
        got = result_dict(bits, r, lab, len(nbr))
        assert_parity(got, oracle_run(nbr, dist, M, eps))
        reused += r.stats["ell_reused"]
        if i == 0:
            assert r.stats["ell_reused"] == 0
    assert reused >= 1, "no call of the sweep reused the ELL"


def test_reuse_request_on_another_graph_rebuilds():
    nbr, dist = _points(5, 2000, 3, 48)
    nbr2, dist2 = _points(6, 2000, 3, 48)
    M = 10
    ws = torch.empty(kdb.workspace_bytes(kdb.Graph(torch.from_numpy(nbr).cuda(), torch.from_numpy(dist).cuda(),
                                                   n_total=2000, exact=True)), dtype=torch.uint8, device="cuda")
    g1 = kdb.Graph(torch.from_numpy(nbr).cuda(), torch.from_numpy(dist).cuda(), n_total=2000, exact=True)
    g2 = kdb.Graph(torch.from_numpy(nbr2).cuda(), torch.from_numpy(dist2).cuda(), n_total=2000, exact=True)
    eps1 = float(eps_from_graph(dist, M, 1.5))
    eps2 = float(eps_from_graph(dist2, M, 1.5))
    kdb.kdbscan(g1, M, eps1, workspace=ws)
    bits, r, lab = kdb.kdbscan(g2, M, eps2, workspace=ws, reuse=True)  # other pointers: must rebuild
    torch.cuda.synchronize()
    assert r.stats["ell_reused"] == 0
    assert_parity(result_dict(bits, r, lab, 2000), oracle_run(nbr2, dist2, M, eps2))
    # same graph, other edge_cols: must rebuild too
    bits, r, lab = kdb.kdbscan(g2, M, eps2, workspace=ws, reuse=True, edge_cols=M)
    torch.cuda.synchronize()
    assert r.stats["ell_reused"] == 0
    assert_parity(result_dict(bits, r, lab, 2000), oracle_run(nbr2, dist2, M, eps2, edge_cols=M))
    # a genuine repeat on the same graph and edge_cols (the light/heavy split,
    # k = 48 >= 40) reuses: first rebuild, then reuse at another eps
    kdb.kdbscan(g2, M, eps2, workspace=ws)
    eps3 = float(eps_from_graph(dist2, M, 1.1))
    bits, r, lab = kdb.kdbscan(g2, M, eps3, workspace=ws, reuse=True)
    torch.cuda.synchronize()
    assert r.stats["ell_reused"] == 1
    assert_parity(result_dict(bits, r, lab, 2000), oracle_run(nbr2, dist2, M, eps3))
