"""GPU <-> oracle parity through the C-ABI (pytest -m gpu).

Bar (north_star): core flags, labels and MSF edge set bit-identical to the
oracle; MSF total weight within 1e-6 relative (the GPU sums exactly and rounds
once, the oracle sums in key order, so they agree far below that).
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

from datagen import eps_from_graph, gen_c1, knn_bruteforce, random_graph
from tests.kdb_harness import assert_parity, oracle_run, run_gpu
from tests.kdb_harness import kdb_opt as _kdb_opt

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2009_04552_b200 as kdb
    kdb.lib()  # fail loudly if the extension is missing


def _golden(name):
    return json.load(open(os.path.join(GOLDEN, name)))


def _golden_cases():
    out = []
    for f in ["w1_fig_cycle.json", "w2_fig_cut_mst.json", "w3_unit_square.json"]:
        g = _golden(f)
        for c in g["cases"]:
            out.append((g["nbr"], g["dist"], c))
        if "dup" in g:
            for c in g["dup"]["cases"]:
                out.append((g["dup"]["nbr"], g["dup"]["dist"], c))
    return out


@pytest.mark.parametrize("idx", range(7))
@pytest.mark.parametrize("P", [0, 1, 2, 3, 4])
def test_golden_examples(idx, P):
    import paper_2009_04552_b200 as kdb
    nbr, dist, case = _golden_cases()[idx]
    nbr = np.array(nbr, np.int32); dist = np.array(dist, np.float32)
    comm = kdb.Comm.sim(P) if P else None
    got = run_gpu(nbr, dist, case["M"], case["eps"], exact=False, comm=comm)
    assert got["core"].tolist() == case["core"]
    assert sorted(zip(got["msf_a"].tolist(), got["msf_b"].tolist())) == sorted(map(tuple, case["msf"]))
    assert got["msf_weight"] == case["msf_weight"]
    assert got["labels"].tolist() == case["labels"]
    assert_parity(got, oracle_run(nbr, dist, case["M"], case["eps"]))


def test_w1_false_exact_promise_is_detected():
    """Fig. cycle's graph is approximate.  Promising EXACT
    for it makes the row-only offers of V2 miss its in-edge from V1, i.e. the
    directed-scan 4-cycle the paper describes; kdb_mst must detect the broken
    promise (a hook target with a larger key) instead of spinning or returning
    a wrong forest."""
    import paper_2009_04552_b200 as kdb
    g = _golden("w1_fig_cycle.json")
    with pytest.raises(kdb.KdbError, match="EXACT"):
        run_gpu(np.array(g["nbr"], np.int32), np.array(g["dist"], np.float32), 1, 0.2, exact=True)


def test_w3_exact_mode():
    g = _golden("w3_unit_square.json")
    for src in (g, g["dup"]):
        for c in src["cases"]:
            nbr = np.array(src["nbr"], np.int32); dist = np.array(src["dist"], np.float32)
            got = run_gpu(nbr, dist, c["M"], c["eps"], exact=True)
            assert_parity(got, oracle_run(nbr, dist, c["M"], c["eps"]))


RANDOM_CASES = [
    # n, k, M, seed, levels, symmetric, pad, zero, local, eps quantile
    (1000, 4, 2, 0, 4, True, 0.0, 0.0, None, 0.6),
    (2000, 8, 3, 1, 3, False, 0.1, 0.05, 30, 0.5),
    (3001, 16, 8, 2, None, True, 0.2, 0.0, None, 0.7),
    (4097, 8, 1, 3, 2, True, 0.0, 0.2, 20, 0.9),
    (5000, 12, 6, 4, 16, False, 0.3, 0.0, 60, 0.4),
    (777, 5, 5, 5, 5, True, 0.0, 0.1, 8, 0.95),
]


@pytest.mark.parametrize("case", RANDOM_CASES)
def test_random_graphs_general(case):
    n, k, M, seed, levels, sym, pad, zero, local, q = case
    nbr, dist = random_graph(n, k, seed, levels=levels, symmetric=sym, pad_frac=pad, zero_frac=zero, local=local)
    fin = dist[np.isfinite(dist)].astype(np.float64)
    eps = np.float32(np.quantile(fin, q))
    exp = oracle_run(nbr, dist, M, eps)
    got = run_gpu(nbr, dist, M, eps, exact=False)
    assert_parity(got, exp)


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_sim_ranks_identical(P):
    import paper_2009_04552_b200 as kdb
    nbr, dist = random_graph(3000, 8, 7, levels=4, symmetric=False, pad_frac=0.1, local=40)
    eps = np.float32(np.quantile(dist[np.isfinite(dist)].astype(np.float64), 0.6))
    exp = oracle_run(nbr, dist, 3, eps)
    got1 = run_gpu(nbr, dist, 3, eps)
    gotP = run_gpu(nbr, dist, 3, eps, comm=kdb.Comm.sim(P))
    assert_parity(got1, exp)
    assert_parity(gotP, exp)
    for key in ("core", "comp", "labels", "msf_a", "msf_b", "msf_w"):
        assert np.array_equal(got1[key], gotP[key])
    assert got1["msf_weight"] == gotP["msf_weight"]


@pytest.fixture(scope="module")
def c1_graph():
    X, _ = gen_c1(0)
    nbr, dist = knn_bruteforce(X, 16)
    return X, nbr, dist


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("P", [0, 4])
def test_config_c1_full(c1_graph, exact, P):
    """BASELINE.json configs[0] at full size: exact kNN graph k=16, M=8,
    eps = 1.5 x median 8th-NN distance."""
    import paper_2009_04552_b200 as kdb
    X, nbr, dist = c1_graph
    eps = eps_from_graph(dist, 8, 1.5)
    exp = oracle_run(nbr, dist, 8, eps)
    got = run_gpu(nbr, dist, 8, eps, exact=exact, comm=kdb.Comm.sim(P) if P else None)
    assert_parity(got, exp)
    assert got["stats"]["rounds"] >= 1


@pytest.mark.parametrize("factor", [0.3, 0.8, 1.0, 2.5, 10.0])
def test_c1_eps_sweep_exact(c1_graph, factor):
    """One graph, many eps (Fig. eps_mnist protocol)."""
    X, nbr, dist = c1_graph
    eps = eps_from_graph(dist, 8, factor)
    exp = oracle_run(nbr, dist, 8, eps)
    assert_parity(run_gpu(nbr, dist, 8, eps, exact=True), exp)


def test_points_exact_graphs_small_k():
    rng = np.random.default_rng(3)
    for t in range(4):
        n = int(rng.integers(50, 2500))
        X = (rng.standard_normal((n, 3)) * rng.uniform(0.1, 1.0)).astype(np.float32)
        X[rng.integers(0, n, n // 20)] = X[rng.integers(0, n, n // 20)]  # duplicates -> w = 0
        k = int(rng.integers(2, 20)); M = int(rng.integers(1, k + 1))
        nbr, dist = knn_bruteforce(X, k)
        eps = eps_from_graph(dist, M, float(rng.uniform(0.8, 3.0)))
        exp = oracle_run(nbr, dist, M, eps)
        assert_parity(run_gpu(nbr, dist, M, eps, exact=True), exp)
        assert_parity(run_gpu(nbr, dist, M, eps, exact=False), exp)


def test_k_full_graph():
    """k = N-1 (the complete graph, Thm. 2(i))."""
    rng = np.random.default_rng(11)
    X = rng.uniform(size=(300, 2)).astype(np.float32)
    nbr, dist = knn_bruteforce(X, 299)
    eps = eps_from_graph(dist, 5, 1.0)
    exp = oracle_run(nbr, dist, 5, eps)
    assert_parity(run_gpu(nbr, dist, 5, eps, exact=True), exp)
    assert_parity(run_gpu(nbr, dist, 5, eps, exact=False), exp)


@pytest.mark.parametrize("n", [1, 2, 3, 33])
def test_degenerate_sizes(n):
    k = max(1, n - 1)
    if n == 1:
        nbr = np.full((1, 1), -1, np.int32); dist = np.full((1, 1), np.inf, np.float32)
    else:
        X = np.random.default_rng(n).uniform(size=(n, 2)).astype(np.float32)
        nbr, dist = knn_bruteforce(X, k)
    for eps in (1e-6, 0.3, 10.0):
        exp = oracle_run(nbr, dist, 1, eps)
        assert_parity(run_gpu(nbr, dist, 1, eps, exact=True), exp)
        assert_parity(run_gpu(nbr, dist, 1, eps), exp)


def test_all_noise_and_all_core():
    nbr, dist = random_graph(500, 6, 1, levels=8)
    exp = oracle_run(nbr, dist, 6, 1e-4)
    got = run_gpu(nbr, dist, 6, 1e-4)
    assert_parity(got, exp)
    assert np.all(got["labels"] == -1) and len(got["msf_a"]) == 0
    exp = oracle_run(nbr, dist, 1, 5.0)
    assert_parity(run_gpu(nbr, dist, 1, 5.0), exp)


def test_determinism_repeat():
    nbr, dist = random_graph(4000, 8, 9, levels=3, symmetric=True, local=25)
    eps = np.float32(0.7)
    a = run_gpu(nbr, dist, 2, eps)
    for _ in range(3):
        b = run_gpu(nbr, dist, 2, eps)
        for key in ("core", "comp", "labels", "msf_a", "msf_b", "msf_w"):
            assert np.array_equal(a[key], b[key])
        assert a["msf_weight"] == b["msf_weight"]


def test_invalid_arguments_raise():
    import paper_2009_04552_b200 as kdb
    nbr, dist = random_graph(64, 4, 0)
    g = kdb.Graph(torch.from_numpy(nbr).cuda(), torch.from_numpy(dist).cuda(), n_total=64)
    with pytest.raises(kdb.KdbError):
        kdb.core_mark(g, 5, 0.5)          # M > k
    with pytest.raises(kdb.KdbError):
        kdb.core_mark(g, 2, 0.0)          # eps not in (0, inf)
    with pytest.raises(kdb.KdbError):
        kdb.core_mark(g, 2, float("inf"))
    bad = kdb.Graph(torch.from_numpy(nbr).cuda(), torch.from_numpy(dist).cuda(), n_total=10)
    with pytest.raises(kdb.KdbError):
        kdb.core_mark(bad, 2, 0.5)        # rows outside [0, N)


# ---- Filter-Boruvka (light phase + filter + heavy phase) ---------
@pytest.mark.parametrize("light", ["1", "2", "3", "6"])
@pytest.mark.parametrize("case", RANDOM_CASES)
def test_random_graphs_filter(case, light, monkeypatch):
    """Light thresholds at several columns: the light MSF + filtered heavy MSF
    must equal Kruskal's MSF of the whole candidate graph on adversarial graphs
    (ties in random id order, asymmetric weights, padding, w = 0)."""
    _kdb_opt("KDB_LIGHT", light)
    n, k, M, seed, levels, sym, pad, zero, local, q = case
    if int(light) >= k:
        pytest.skip("light column beyond k")
    nbr, dist = random_graph(n, k, seed, levels=levels, symmetric=sym, pad_frac=pad, zero_frac=zero, local=local)
    eps = np.float32(np.quantile(dist[np.isfinite(dist)].astype(np.float64), q))
    got = run_gpu(nbr, dist, M, eps, exact=False)
    assert_parity(got, oracle_run(nbr, dist, M, eps))


@pytest.mark.parametrize("light", ["2", "4", "8"])
@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("P", [0, 3])
def test_c1_filter(c1_graph, light, exact, P, monkeypatch):
    import paper_2009_04552_b200 as kdb
    _kdb_opt("KDB_LIGHT", light)
    X, nbr, dist = c1_graph
    eps = eps_from_graph(dist, 8, 1.5)
    got = run_gpu(nbr, dist, 8, eps, exact=exact, comm=kdb.Comm.sim(P) if P else None)
    assert_parity(got, oracle_run(nbr, dist, 8, eps))
    st = got["stats"]
    assert st["tau"] >= 0 and st["fallback"] == 0, st  # the filter path really ran
    assert st["light_components"] >= 1


def test_filter_overflow_falls_back(c1_graph, monkeypatch):
    """A survivor buffer too small for the crossing heavy entries: kdb_mst
    reruns plain rows-Boruvka and the result is still exact."""
    _kdb_opt("KDB_LIGHT", "2")
    _kdb_opt("KDB_SURVCAP", "0")
    X, nbr, dist = c1_graph
    eps = eps_from_graph(dist, 8, 1.5)
    got = run_gpu(nbr, dist, 8, eps, exact=True)
    assert_parity(got, oracle_run(nbr, dist, 8, eps))
    assert got["stats"]["fallback"] == 1 and got["stats"]["survivors"] > 0


def test_filter_off_matches(c1_graph, monkeypatch):
    _kdb_opt("KDB_FILTER", "0")
    X, nbr, dist = c1_graph
    eps = eps_from_graph(dist, 8, 1.5)
    got = run_gpu(nbr, dist, 8, eps, exact=True)
    assert_parity(got, oracle_run(nbr, dist, 8, eps))
    assert got["stats"]["tau"] == -1.0


@pytest.mark.parametrize("light", ["1", "3", "10"])
def test_points_filter_exact_graphs(light, monkeypatch):
    _kdb_opt("KDB_LIGHT", light)
    rng = np.random.default_rng(int(light))
    for t in range(3):
        n = int(rng.integers(200, 3000))
        X = (rng.standard_normal((n, 3)) * rng.uniform(0.1, 1.0)).astype(np.float32)
        X[rng.integers(0, n, n // 20)] = X[rng.integers(0, n, n // 20)]
        k = int(rng.integers(12, 24)); M = int(rng.integers(1, k + 1))
        nbr, dist = knn_bruteforce(X, k)
        eps = eps_from_graph(dist, M, float(rng.uniform(0.8, 3.0)))
        exp = oracle_run(nbr, dist, M, eps)
        for P in (0, 2):
            import paper_2009_04552_b200 as kdb
            comm = kdb.Comm.sim(P) if P else None
            assert_parity(run_gpu(nbr, dist, M, eps, exact=True, comm=comm), exp)
            assert_parity(run_gpu(nbr, dist, M, eps, exact=False, comm=comm), exp)


@pytest.fixture(scope="module")
def c4_small_graph():
    """The C4 recipe at 128K points (10 spheres, exact grid kNN graph k = 100) and
    the oracle's result at the config's eps rule."""
    from datagen import CONFIGS, gen_config_points
    from paper_2009_04552_b200.knng import build_knng_grid
    X, _ = gen_config_points("C4", 0, 0.002)
    nbr_t, dist_t, _ = build_knng_grid(X, 100, device="cuda")
    nbr, dist = nbr_t.cpu().numpy(), dist_t.cpu().numpy()
    eps = float(np.float32(CONFIGS["C4"]["eps_factor"] * float(np.median(dist[:, 49].astype(np.float64)))))
    return nbr, dist, eps, oracle_run(nbr, dist, 50, eps)


@pytest.mark.parametrize("knob", ["KDB_LVL", "KDB_LVL=2", "KDB_LVL=3", "KDB_QUAD", "KDB_REFILL", "KDB_LEAN", "KDB_FASTSCAN", "KDB_TILE"])
def test_light_round_variants_kept_off(knob, c4_small_graph, monkeypatch):
    """The light-round variants that were measured slower and are off by default
    (DESIGN.md section 16 and its options table) stay parity-green on the path the
    bench runs (one rank, exact graph, light split): the C4 recipe at 128K points,
    and small clustered point sets with duplicate points (ties, w = 0)."""
    _kdb_opt(knob.split("=")[0], knob.split("=")[1] if "=" in knob else "1")
    nbr, dist, eps, exp = c4_small_graph
    assert_parity(run_gpu(nbr, dist, 50, eps, exact=True), exp)
    _kdb_opt("KDB_LIGHT", "6")
    rng = np.random.default_rng(len(knob))
    for t in range(3):
        n = int(rng.integers(1000, 5000))
        X = (rng.standard_normal((n, 3)) * rng.uniform(0.1, 1.0)).astype(np.float32)
        X[rng.integers(0, n, n // 20)] = X[rng.integers(0, n, n // 20)]
        k = int(rng.integers(12, 24)); M = int(rng.integers(1, k + 1))
        nbr2, dist2 = knn_bruteforce(X, k)
        eps2 = eps_from_graph(dist2, M, float(rng.uniform(0.8, 3.0)))
        assert_parity(run_gpu(nbr2, dist2, M, eps2, exact=True), oracle_run(nbr2, dist2, M, eps2))


@pytest.mark.parametrize("filt", ["0", "1"])
@pytest.mark.parametrize("case", RANDOM_CASES)
def test_inplace_rows_mode(case, filt, monkeypatch):
    """KDB_COMPACT=0: the rows phase reads the graph rows in place instead of
    the compact light lists (the path taken when the lists exceed capacity)."""
    _kdb_opt("KDB_COMPACT", "0")
    _kdb_opt("KDB_FILTER", filt)
    _kdb_opt("KDB_LIGHT", "2")
    n, k, M, seed, levels, sym, pad, zero, local, q = case
    nbr, dist = random_graph(n, k, seed, levels=levels, symmetric=sym, pad_frac=pad, zero_frac=zero, local=local)
    eps = np.float32(np.quantile(dist[np.isfinite(dist)].astype(np.float64), q))
    assert_parity(run_gpu(nbr, dist, M, eps, exact=False), oracle_run(nbr, dist, M, eps))


@pytest.mark.parametrize("exact", [False, True])
def test_c1_inplace_rows_mode(c1_graph, exact, monkeypatch):
    _kdb_opt("KDB_COMPACT", "0")
    X, nbr, dist = c1_graph
    eps = eps_from_graph(dist, 8, 1.5)
    for P in (0, 2):
        import paper_2009_04552_b200 as kdb
        got = run_gpu(nbr, dist, 8, eps, exact=exact, comm=kdb.Comm.sim(P) if P else None)
        assert_parity(got, oracle_run(nbr, dist, 8, eps))


@pytest.mark.parametrize("fast", ["0", "1"])
@pytest.mark.parametrize("light", ["2", "4"])
def test_filter_fast_path_toggle(c1_graph, fast, light, monkeypatch):
    """The filter's shared-memory fast path (dominant component per id block +
    Bloom filter of the exceptions) must give the same survivors as the plain
    per-entry gather; shuffled ids (no block locality) exercise its slow path."""
    _kdb_opt("KDB_FASTFILTER", fast)
    _kdb_opt("KDB_LIGHT", light)
    X, nbr, dist = c1_graph
    eps = eps_from_graph(dist, 8, 1.5)
    got = run_gpu(nbr, dist, 8, eps, exact=True)
    assert_parity(got, oracle_run(nbr, dist, 8, eps))
    # the same point set under a random id permutation
    n = len(X)
    perm = np.random.default_rng(5).permutation(n)
    Xp = X[perm]
    nbr2, dist2 = knn_bruteforce(Xp, 16)
    eps2 = eps_from_graph(dist2, 8, 1.5)
    got2 = run_gpu(nbr2, dist2, 8, eps2, exact=True)
    assert_parity(got2, oracle_run(nbr2, dist2, 8, eps2))


@pytest.mark.parametrize("k", [20, 24, 28, 37, 100, 130])
def test_wide_rows_exact(k):
    """k % 4 == 0 and k >= 20: the light ELL is read with 32-byte sector loads
    (rows start at a 32-B boundary or 16 B past one)."""
    rng = np.random.default_rng(k)
    n = 3000
    X = np.concatenate([rng.standard_normal((n // 2, 3)) * 0.05, rng.standard_normal((n - n // 2, 3)) * 0.05 + 1.0])
    X = X.astype(np.float32)
    nbr, dist = knn_bruteforce(X, k)
    for M, f in ((k // 2, 1.5), (5, 1.0)):
        eps = eps_from_graph(dist, M, f)
        exp = oracle_run(nbr, dist, M, eps)
        assert_parity(run_gpu(nbr, dist, M, eps, exact=True), exp)
        assert_parity(run_gpu(nbr, dist, M, eps, exact=False), exp)


@pytest.mark.parametrize("k", [1028, 1030])
def test_very_wide_rows_filter_division(k):
    """Rows of >= 1,024 entries: the filter's entry -> row division inside a
    4,096-row tile leaves the 32-bit multiply-high path (exact only for
    n * d < 2^32) for the 64-bit one; VEC 4 (k % 4 == 0) and VEC 1."""
    rng = np.random.default_rng(k)
    n = 2500
    X = np.concatenate([rng.standard_normal((n // 2, 3)) * 0.05, rng.standard_normal((n - n // 2, 3)) * 0.05 + 1.0])
    X = X.astype(np.float32)
    nbr, dist = knn_bruteforce(X, k)
    for M, f in ((k // 2, 1.5), (5, 1.0)):
        eps = eps_from_graph(dist, M, f)
        exp = oracle_run(nbr, dist, M, eps)
        assert_parity(run_gpu(nbr, dist, M, eps, exact=True), exp)
        assert_parity(run_gpu(nbr, dist, M, eps, exact=False), exp)


@pytest.mark.parametrize("fuse,pack", [("0", "0"), ("1", "0"), ("1", "1")])
@pytest.mark.parametrize("P", [0, 3])
def test_round1_fused_into_ell(c1_graph, fuse, pack, P, monkeypatch):
    """Exact mode: round 1 (singleton components) computed inside the light-ELL
    pass (KDB_FUSE1=1, default) or by its own kernel (0); on a single rank the
    round-1 hook reads one packed (K, B, kmin) record per component
    (KDB_PACK1=1, default) -- same forest."""
    import paper_2009_04552_b200 as kdb
    _kdb_opt("KDB_FUSE1", fuse)
    _kdb_opt("KDB_PACK1", pack)
    X, nbr, dist = c1_graph
    for M, f in ((8, 1.5), (3, 0.7), (12, 3.0)):
        eps = eps_from_graph(dist, M, f)
        got = run_gpu(nbr, dist, M, eps, exact=True, comm=kdb.Comm.sim(P) if P else None)
        assert_parity(got, oracle_run(nbr, dist, M, eps))





@pytest.mark.parametrize("sparse", ["0", "1"])
@pytest.mark.parametrize("case", RANDOM_CASES)
def test_sparse_ids_toggle(case, sparse, monkeypatch):
    """Late rounds keep root ids (no dense renumbering) -- same bits either way,
    general and exact mode, filtered and unfiltered."""
    _kdb_opt("KDB_SPARSE", sparse)
    n, k, M, seed, levels, sym, pad, zero, local, q = case
    nbr, dist = random_graph(n, k, seed, levels=levels, symmetric=sym, pad_frac=pad, zero_frac=zero, local=local)
    eps = np.float32(np.quantile(dist[np.isfinite(dist)].astype(np.float64), q))
    exp = oracle_run(nbr, dist, M, eps)
    for filt in ("0", "1"):
        _kdb_opt("KDB_FILTER", filt)
        assert_parity(run_gpu(nbr, dist, M, eps, exact=False), exp)


@pytest.mark.parametrize("sparse", ["0", "1"])
@pytest.mark.parametrize("P", [0, 3])
def test_c1_sparse_ids(c1_graph, sparse, P, monkeypatch):
    import paper_2009_04552_b200 as kdb
    _kdb_opt("KDB_SPARSE", sparse)
    X, nbr, dist = c1_graph
    for exact in (False, True):
        for f in (1.0, 1.5, 3.0):
            eps = eps_from_graph(dist, 8, f)
            got = run_gpu(nbr, dist, 8, eps, exact=exact, comm=kdb.Comm.sim(P) if P else None)
            assert_parity(got, oracle_run(nbr, dist, 8, eps))


@pytest.mark.parametrize("exact", [False, True])
def test_nccl_communicator_one_rank(c1_graph, exact, monkeypatch):
    """A real NCCL communicator (1 rank; KDB_NCCL_FORCE=1 issues every collective
    anyway): the multi-rank host logic -- exact per-round counts (sync_each),
    all-reduced core bits / keys / ties / targets / tau / overflow branch, the
    heavy-phase exchanges -- runs through NCCL on one GPU and gives the oracle's
    result."""
    import ctypes as C
    import paper_2009_04552_b200 as kdb
    _kdb_opt("KDB_NCCL_FORCE", "1")
    b = (C.c_ubyte * 128)()
    assert kdb.lib().kdb_nccl_unique_id(C.cast(b, C.c_void_p)) == 0
    h = C.c_void_p()
    assert kdb.lib().kdb_comm_create_nccl(C.byref(h), C.cast(b, C.c_void_p), 0, 1) == 0
    comm = kdb.Comm(h, 1, 0, "nccl")  # == kdb.Comm.nccl_single()
    X, nbr, dist = c1_graph
    try:
        for light in ("2", "10"):
            _kdb_opt("KDB_LIGHT", light)
            for f in (1.0, 1.5):
                eps = eps_from_graph(dist, 8, f)
                assert_parity(run_gpu(nbr, dist, 8, eps, exact=exact, comm=comm), oracle_run(nbr, dist, 8, eps))
    finally:
        comm.close()


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_narrow_rows(k):
    """Rows narrower than the light ELL (kW = 16) and than one 4-entry chunk;
    M = k and M = 1; general and exact mode; sim ranks."""
    import paper_2009_04552_b200 as kdb
    rng = np.random.default_rng(100 + k)
    X = rng.standard_normal((1500, 2)).astype(np.float32)
    nbr, dist = knn_bruteforce(X, k)
    for M in sorted({1, k}):
        for f in (1.0, 3.0):
            eps = eps_from_graph(dist, M, f)
            exp = oracle_run(nbr, dist, M, eps)
            for exact in (False, True):
                assert_parity(run_gpu(nbr, dist, M, eps, exact=exact), exp)
            assert_parity(run_gpu(nbr, dist, M, eps, comm=kdb.Comm.sim(3)), exp)


@pytest.mark.parametrize("pre", ["0", "1"])
@pytest.mark.parametrize("case", RANDOM_CASES)
def test_offer_precheck_toggle(case, pre, monkeypatch):
    """Offers read the current key before their atomicMin (KDB_PRECHECK forces
    it on / off; by default it switches on once live rows outnumber the
    components 8 to 1) -- the same forest either way, in every round kernel."""
    _kdb_opt("KDB_PRECHECK", pre)
    n, k, M, seed, levels, sym, pad, zero, local, q = case
    nbr, dist = random_graph(n, k, seed, levels=levels, symmetric=sym, pad_frac=pad, zero_frac=zero, local=local)
    eps = np.float32(np.quantile(dist[np.isfinite(dist)].astype(np.float64), q))
    exp = oracle_run(nbr, dist, M, eps)
    for compact in ("0", "1"):
        _kdb_opt("KDB_COMPACT", compact)
        assert_parity(run_gpu(nbr, dist, M, eps, exact=False), exp)


@pytest.mark.parametrize("L", [7, 30])
@pytest.mark.parametrize("P", [0, 3])
def test_torus_ties_force_the_sweep_round(L, P):
    """L x L torus, k = 4: every row holds its 4 lattice neighbours at w = 1, so
    kth'(v) = 1 equals every offer and no component can certify (reading #20):
    the exact mode must stall and finish with edge-centric sweep rounds.  The
    graph is an exact kNN graph of the torus metric (symmetric, mirrored)."""
    import paper_2009_04552_b200 as kdb
    n = L * L
    ids = np.arange(n).reshape(L, L)
    nb = np.stack([np.roll(ids, 1, 0), np.roll(ids, -1, 0), np.roll(ids, 1, 1), np.roll(ids, -1, 1)], -1)
    nbr = nb.reshape(n, 4).astype(np.int32)
    dist = np.ones((n, 4), np.float32)
    exp = oracle_run(nbr, dist, 4, 1.0)
    got = run_gpu(nbr, dist, 4, 1.0, exact=True, comm=kdb.Comm.sim(P) if P else None)
    assert_parity(got, exp)
    assert got["stats"]["stall_rounds"] > 0
    assert len(exp["msf_a"]) == n - 1
    assert_parity(run_gpu(nbr, dist, 4, 1.0, exact=False), exp)


@pytest.mark.parametrize("pipe", ["0", "1"])
@pytest.mark.parametrize("case", RANDOM_CASES)
def test_pipelined_chunk_loads_toggle(case, pipe, monkeypatch):
    """scan_ell with the next ELL chunk's load issued ahead (KDB_PIPE forces it
    on / off; by default it follows the share of all-light ELL rows)."""
    _kdb_opt("KDB_PIPE", pipe)
    n, k, M, seed, levels, sym, pad, zero, local, q = case
    nbr, dist = random_graph(n, k, seed, levels=levels, symmetric=sym, pad_frac=pad, zero_frac=zero, local=local)
    eps = np.float32(np.quantile(dist[np.isfinite(dist)].astype(np.float64), q))
    exp = oracle_run(nbr, dist, M, eps)
    for light in ("2", "10"):
        _kdb_opt("KDB_LIGHT", light)
        assert_parity(run_gpu(nbr, dist, M, eps, exact=False), exp)


@pytest.mark.parametrize("n", [40, 5000, 50000])
def test_star_forest_hub_runs(n):
    """Every vertex's nearest neighbour is vertex 0: the MSF is a star, one run
    of n-1 edges with a = 0.  Runs longer than kRunMax are sorted by the
    segmented sort (an insertion sort per run was quadratic: 220 s at 1e5)."""
    import time
    k = 4
    rng = np.random.default_rng(n)
    nbr = np.empty((n, k), np.int32)
    dist = np.empty((n, k), np.float32)
    nbr[0] = np.arange(1, k + 1)
    dist[0] = 0.1
    others = rng.integers(1, n, size=(n, k - 1)).astype(np.int32)
    v = np.arange(n, dtype=np.int32)[:, None]
    others = np.where(others == v, (v % (n - 1)) + 1, others).astype(np.int32)  # no self entries
    nbr[1:, 0] = 0
    nbr[1:, 1:] = others[1:]
    dist[1:] = [0.1, 0.5, 0.6, 0.7]
    exp = oracle_run(nbr, dist, 1, 1.0)
    t = time.time()
    got = run_gpu(nbr, dist, 1, 1.0, exact=False)
    assert time.time() - t < 5.0
    assert_parity(got, exp)
    assert np.all(got["msf_a"] == 0) and len(got["msf_a"]) == n - 1


@pytest.mark.parametrize("skip", ["0", "1"])
@pytest.mark.parametrize("P", [0, 3])
def test_round2_head_skip_toggle(c1_graph, skip, P, monkeypatch):
    """Round-2 heads start past the entry a certified singleton hooked along
    (KDB_SKIP1=1, default) or at it (0): the same forest either way, including
    ties (few weight levels) and the local-first phase under sim ranks."""
    import paper_2009_04552_b200 as kdb
    _kdb_opt("KDB_SKIP1", skip)
    X, nbr, dist = c1_graph
    for f in (0.7, 1.5):
        eps = eps_from_graph(dist, 8, f)
        got = run_gpu(nbr, dist, 8, eps, exact=True, comm=kdb.Comm.sim(P) if P else None)
        assert_parity(got, oracle_run(nbr, dist, 8, eps))
    rng = np.random.default_rng(11)
    X = np.round(rng.uniform(0, 30, size=(1500, 2))).astype(np.float32)  # lattice: many equal distances
    X += (rng.uniform(size=X.shape) < 0.02) * 0.5
    nbr, dist = knn_bruteforce(X, 12)
    eps = eps_from_graph(dist, 4, 1.2)
    got = run_gpu(nbr, dist, 4, eps, exact=True, comm=kdb.Comm.sim(P) if P else None)
    assert_parity(got, oracle_run(nbr, dist, 4, eps))
