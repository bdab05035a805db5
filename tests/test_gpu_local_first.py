"""Local-first contraction (multi-rank exact mode; SURVEY.md
§8(e)(ii)) against the oracle through the C-ABI (pytest -m gpu).

Every rank first contracts its own rows with no exchange -- a component hooks
only along a certified minimum that stays inside the rank (cut property: an MSF
edge whatever the other ranks hold) -- and the components left are finished by
the exchanged rounds.  Thm. 3 says the clusters do not
depend on the partition; here the FOREST must not either: every case is
bit-identical to the oracle for every rank count, and to the run with the
local phase switched off (KDB_LOCAL=0).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from datagen import eps_from_graph, gen_c1, knn_bruteforce
from tests.kdb_harness import assert_parity, oracle_run, run_gpu
from tests.kdb_harness import kdb_opt as _kdb_opt

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1_graph():
    X, _ = gen_c1(0)
    nbr, dist = knn_bruteforce(X, 16)
    return nbr, dist


@pytest.mark.parametrize("P", [2, 3, 5, 8])
@pytest.mark.parametrize("light", ["2", "10", "off"])
def test_c1_local_first(c1_graph, P, light, monkeypatch):
    import paper_2009_04552_b200 as kdb
    nbr, dist = c1_graph
    if light == "off":
        _kdb_opt("KDB_FILTER", "0")
    else:
        _kdb_opt("KDB_LIGHT", light)
    for f in (0.6, 1.5, 4.0):
        eps = eps_from_graph(dist, 8, f)
        exp = oracle_run(nbr, dist, 8, eps)
        got = run_gpu(nbr, dist, 8, eps, exact=True, comm=kdb.Comm.sim(P))
        assert_parity(got, exp)
        lf = got["stats"].get("local_first")
        assert lf is not None and lf["local_ms_sum"] >= lf["local_ms_max"] >= 0
        assert 0 <= lf["parked_rows"] <= len(nbr)
        _kdb_opt("KDB_LOCAL", "0")
        off = run_gpu(nbr, dist, 8, eps, exact=True, comm=kdb.Comm.sim(P))
        kdb.reset_options()
        assert "local_first" not in off["stats"]
        assert_parity(off, exp)


def _clustered(seed, n, d=3, n_noise=0):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-4, 4, size=(6, d))
    X = c[rng.integers(0, 6, n)] + 0.35 * rng.standard_normal((n, d))
    if n_noise:
        X = np.concatenate([X, rng.uniform(-60, 60, size=(n_noise, d))])
    return X.astype(np.float32)


@pytest.mark.parametrize("seed", range(4))
def test_points_local_first(seed):
    import paper_2009_04552_b200 as kdb
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(300, 3000))
    X = _clustered(seed, n)
    X[rng.integers(0, n, n // 25)] = X[rng.integers(0, n, n // 25)]  # duplicates: w = 0 ties
    k = int(rng.integers(4, 24)); M = int(rng.integers(1, k + 1))
    nbr, dist = knn_bruteforce(X, k)
    for f in (0.9, 2.0):
        eps = eps_from_graph(dist, M, f)
        exp = oracle_run(nbr, dist, M, eps)
        for P in (2, 4, 7):
            assert_parity(run_gpu(nbr, dist, M, eps, exact=True, comm=kdb.Comm.sim(P)), exp)


def test_rank_without_core_rows():
    """The last ranks hold only far-away noise rows (no core row, nothing to
    contract locally); their rows still take part in the border pass."""
    import paper_2009_04552_b200 as kdb
    X = _clustered(7, 800, n_noise=400)
    nbr, dist = knn_bruteforce(X, 12)
    eps = eps_from_graph(dist[:800], 6, 1.5)
    exp = oracle_run(nbr, dist, 6, eps)
    assert exp["core"][800:].sum() == 0 and exp["core"][:800].sum() > 0
    for P in (3, 6):
        got = run_gpu(nbr, dist, 6, eps, exact=True, comm=kdb.Comm.sim(P))
        assert_parity(got, exp)


@pytest.mark.parametrize("scale", [0.002])
def test_c4_recipe_local_first(scale):
    """The C4 recipe at 128K points (10 spheres, exact grid kNN graph k = 100):
    the clusters straddle rank boundaries at P = 8 (ids are random inside a
    cluster), so most of a straddling cluster's rows freeze on remote minima and
    finish in the global phase -- which must still give the oracle's forest."""
    import paper_2009_04552_b200 as kdb
    from datagen import CONFIGS, gen_config_points
    from paper_2009_04552_b200.knng import build_knng_grid
    X, _ = gen_config_points("C4", 0, scale)
    nbr_t, dist_t, _ = build_knng_grid(X, 100, device="cuda")
    nbr, dist = nbr_t.cpu().numpy(), dist_t.cpu().numpy()
    med = float(np.median(dist[:, 49].astype(np.float64)))
    eps = float(np.float32(CONFIGS["C4"]["eps_factor"] * med))
    exp = oracle_run(nbr, dist, 50, eps)
    for P in (2, 4, 8):
        got = run_gpu(nbr, dist, 50, eps, exact=True, comm=kdb.Comm.sim(P))
        assert_parity(got, exp)
        lf = got["stats"]["local_first"]
        assert lf["global_components"] >= 0 and lf["local_rounds"] >= 1
