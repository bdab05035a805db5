"""GPU kNN-graph builders (input construction, separately timed; north_star:
'spot-checked against brute force on sampled rows') against the CPU fp64
brute force of datagen/knn_cpu.py, row for row (pytest -m gpu)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from datagen import gen_c1, knn_bruteforce, knn_rows_bruteforce
from paper_2009_04552_b200.knng import build_knng_brute, build_knng_grid

pytestmark = pytest.mark.gpu


def _same(g_nbr, g_dist, c_nbr, c_dist):
    assert np.array_equal(g_nbr, c_nbr)
    assert np.array_equal(g_dist.view(np.uint32), c_dist.view(np.uint32))


@pytest.mark.parametrize("d", [2, 3, 5])
def test_grid_builder_matches_bruteforce(d):
    rng = np.random.default_rng(d)
    X = rng.uniform(size=(3000, d)).astype(np.float32)
    X[rng.integers(0, 3000, 60)] = X[rng.integers(0, 3000, 60)]  # duplicates: w = 0 and index ties
    nbr, dist, _ = build_knng_grid(X, 20)
    c_nbr, c_dist = knn_bruteforce(X, 20)
    _same(nbr.cpu().numpy(), dist.cpu().numpy(), c_nbr, c_dist)


@pytest.mark.parametrize("d,k,margin", [(10, 100, 32), (50, 32, 32), (7, 16, 0), (50, 32, 1)])
def test_brute_builder_matches_bruteforce(d, k, margin):
    """margin 0/1 forces certificate failures: the exact fallback rows must agree too."""
    rng = np.random.default_rng(d + k)
    n = 4000
    C = rng.standard_normal((4, d)) * 0.2
    X = (C[rng.integers(0, 4, n)] + 0.01 * rng.standard_normal((n, d))).astype(np.float32)
    X[rng.integers(0, n, 40)] = X[rng.integers(0, n, 40)]
    nbr, dist, info = build_knng_brute(X, k, margin=margin)
    c_nbr, c_dist = knn_bruteforce(X, k)
    _same(nbr.cpu().numpy(), dist.cpu().numpy(), c_nbr, c_dist)
    if margin == 0:
        assert info["certificate_failures"] > 0


def test_c1_graph_both_builders():
    X, _ = gen_c1(0)
    a_nbr, a_dist, _ = build_knng_grid(X, 16)
    b_nbr, b_dist, _ = build_knng_brute(X, 16)
    c_nbr, c_dist = knn_bruteforce(X, 16)
    _same(a_nbr.cpu().numpy(), a_dist.cpu().numpy(), c_nbr, c_dist)
    _same(b_nbr.cpu().numpy(), b_dist.cpu().numpy(), c_nbr, c_dist)


def test_torch_spot_checker_matches_cpu_bruteforce():
    """The GPU spot checker (tests/knn_spot.py) is the CPU brute force's definition."""
    from tests.knn_spot import knn_rows_torch
    rng = np.random.default_rng(7)
    X = rng.uniform(size=(5000, 5)).astype(np.float32)
    X[rng.integers(0, 5000, 50)] = X[rng.integers(0, 5000, 50)]
    rows = np.sort(rng.choice(5000, 300, replace=False))
    c_nbr, c_dist = knn_rows_bruteforce(X, rows, 24)
    g_nbr, g_dist = knn_rows_torch(torch.from_numpy(X).cuda(), torch.from_numpy(rows).cuda(), 24, p_chunk=1500)
    _same(g_nbr.cpu().numpy(), g_dist.cpu().numpy(), c_nbr, c_dist)


@pytest.mark.parametrize("name,P", [("C4", 3), ("C5", 4)])
def test_grid_rank_rows_equal_full_graph_rows(name, P):
    """knng_grid_rows: each rank's rows (every point a candidate) are exactly the
    corresponding rows of the whole graph."""
    from datagen import CONFIGS, gen_config_points
    X, _ = gen_config_points(name, 0, 0.005)
    k = CONFIGS[name]["k"]
    nbr, dist, info = build_knng_grid(X, k)
    n = len(X)
    for r in range(P):
        b, e = n * r // P, n * (r + 1) // P
        rn, rd, _ = build_knng_grid(X, k, h=info["h"], rows=(b, e))
        assert torch.equal(rn, nbr[b:e]) and torch.equal(rd.view(torch.int32), dist[b:e].view(torch.int32))


def _spot(X, nbr, dist, row_begin, n_samples, k, truth=None, seed=0):
    """n_samples random rows of the graph against the fp64 brute force; with
    `truth` (C4 / C5: separated unit spheres) each query's candidates are its own
    cluster, after checking that no other cluster can come within the largest
    sampled k-th distance (tests/knn_spot.separated_clusters)."""
    from tests.knn_spot import knn_rows_torch, separated_clusters
    g = torch.Generator(device="cpu").manual_seed(seed)
    loc = torch.randperm(nbr.shape[0], generator=g)[:n_samples].sort().values
    Xd = torch.as_tensor(X).cuda() if isinstance(X, np.ndarray) else X
    l = loc.cuda()
    if truth is None:
        e_nbr, e_dist = knn_rows_torch(Xd, l + row_begin, k)
    else:
        assert separated_clusters(Xd, truth, float(dist[l, k - 1].max()))
        t = np.asarray(truth)
        q = (loc + row_begin).numpy()
        e_nbr = torch.empty((len(q), k), dtype=torch.int32, device="cuda")
        e_dist = torch.empty((len(q), k), dtype=torch.float32, device="cuda")
        for c in np.unique(t[q]):
            sel = np.flatnonzero(t[q] == c)
            ids = np.flatnonzero(t == c)
            en, ed = knn_rows_torch(Xd, torch.from_numpy(q[sel]).cuda(), k, cand=(int(ids[0]), int(ids[-1]) + 1))
            e_nbr[torch.from_numpy(sel).cuda()] = en
            e_dist[torch.from_numpy(sel).cuda()] = ed
    assert torch.equal(nbr[l], e_nbr), "sampled rows: neighbour ids differ from fp64 brute force"
    assert torch.equal(dist[l].view(torch.int32), e_dist.view(torch.int32)), "sampled rows: distances differ"


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_full_size_graph_spot_check(name):
    """10^4 sampled rows of the FULL-size graph of each single-GPU config against
    the fp64 brute force (north_star: "spot-checked against brute force on
    sampled rows")."""
    from datagen import CONFIGS, gen_config_points
    X, truth = gen_config_points(name, 0, 1.0)
    k = CONFIGS[name]["k"]
    build = build_knng_grid if X.shape[1] <= 5 else build_knng_brute
    nbr, dist, _ = build(X, k)
    _spot(X, nbr, dist, 0, 10_000, k, truth=truth if name == "C4" else None)


def test_c5_full_size_rank_rows_spot_check():
    """C5 at full size (256M points, 5-D): rank 3 of 8 builds only its rows
    (knng_grid_rows over all points, the multi-GPU bench's construction); 10^4
    sampled rows against the fp64 brute force."""
    from datagen import CONFIGS, gen_config_points
    X, truth = gen_config_points("C5", 0, 1.0)
    n, k = len(X), CONFIGS["C5"]["k"]
    b, e = n * 3 // 8, n * 4 // 8
    Xd = torch.from_numpy(X).cuda()
    del X
    nbr, dist, _ = build_knng_grid(Xd, k, rows=(b, e))
    _spot(Xd, nbr, dist, b, 10_000, k, truth=truth)
