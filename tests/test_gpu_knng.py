"""GPU kNN-graph builders (input construction, separately timed; north_star:
'spot-checked against brute force on sampled rows') against the CPU fp64
brute force of datagen/knn_cpu.py, row for row (pytest -m gpu)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from datagen import gen_c1, knn_bruteforce, knn_rows_bruteforce
from datagen.knng_gpu import build_knng_brute, build_knng_grid

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
