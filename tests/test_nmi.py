"""Pins for the NMI / cluster-count oracle (oracle/nmi.py; -m "not gpu") and,
with a GPU, parity of kdb_nmi against it (-m gpu)."""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from oracle import nmi as onmi


def test_spec_examples():
    # SPEC.md:425-428 worked examples
    a = np.array([0, 0, 1, 1, 2, 2])
    assert onmi.nmi(a, a) == pytest.approx(1.0, abs=1e-12)
    assert onmi.nmi(np.zeros(6, int), np.array([0, 0, 0, 1, 1, 1])) == 0.0
    assert onmi.nmi(np.array([0, 0, 1, 1]), np.array([0, 1, 0, 1])) == pytest.approx(0.0, abs=1e-15)
    assert onmi.cluster_count(np.full(5, -1)) == 0
    assert onmi.cluster_count(np.array([0, 0, 5, 5, -1])) == 2


def test_hand_computed_table():
    """a = {0,0,1,1}, b = {0,0,0,1}: H(a) = ln 2, H(b) = -(3/4 ln 3/4 + 1/4 ln 1/4),
    I = 1/2 ln 2 + 1/4 ln(1/4 / (1/2 * 3/4)) + 1/4 ln(1/4 / (1/2 * 1/4))."""
    Ha = math.log(2)
    Hb = -(0.75 * math.log(0.75) + 0.25 * math.log(0.25))
    I = 0.5 * math.log(0.5 / (0.5 * 0.75)) + 0.25 * math.log(0.25 / (0.5 * 0.75)) + 0.25 * math.log(0.25 / (0.5 * 0.25))
    exp = 2 * I / (Ha + Hb)
    assert onmi.nmi([0, 0, 1, 1], [0, 0, 0, 1]) == pytest.approx(exp, rel=1e-14)


@pytest.mark.parametrize("seed", range(5))
def test_matches_sklearn_and_invariances(seed):
    from sklearn.metrics import normalized_mutual_info_score as sk
    rng = np.random.default_rng(seed)
    n = 2000
    a = rng.integers(-1, 6, n)
    b = np.where(rng.random(n) < 0.7, a, rng.integers(-1, 9, n))
    v = onmi.nmi(a, b)
    assert v == pytest.approx(sk(a, b, average_method="arithmetic"), abs=1e-12)
    assert onmi.nmi(b, a) == pytest.approx(v, abs=1e-14)                        # symmetry
    perm = rng.permutation(20) + 100
    assert onmi.nmi(np.where(a >= 0, perm[a], -1), b) == pytest.approx(v, abs=1e-14)  # relabelling
    assert 0.0 <= v <= 1.0


def test_noise_is_one_pseudo_cluster():
    # all noise vs all noise: identical single-cluster partitions -> 1
    assert onmi.nmi(np.full(4, -1), np.full(4, -1)) == 1.0
    # noise grouped as one cluster: a partition with noise equals the one with a label in its place
    a = np.array([-1, -1, 0, 0, 1])
    assert onmi.nmi(a, np.array([7, 7, 0, 0, 1])) == pytest.approx(1.0, abs=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("n,ka,kb,noise", [(1, 1, 1, 0.0), (1000, 3, 5, 0.1), (200_000, 50, 7, 0.2),
                                            (300_001, 3000, 3000, 0.0), (50_000, 1, 4, 0.5)])
def test_kdb_nmi_parity(n, ka, kb, noise):
    import paper_2009_04552_b200 as kdb
    rng = np.random.default_rng(n)
    a = rng.integers(0, ka, n).astype(np.int32)
    b = np.where(rng.random(n) < 0.6, a % kb, rng.integers(0, kb, n)).astype(np.int32)
    a[rng.random(n) < noise] = -1
    b[rng.random(n) < noise / 2] = -1
    v, ca, cb = kdb.nmi(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    exp = onmi.nmi(a, b)
    assert v == pytest.approx(exp, abs=1e-9)
    assert ca == onmi.cluster_count(a) and cb == onmi.cluster_count(b)
