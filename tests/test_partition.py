"""The inertial point order (datagen/partition.py; "we partition the
datasets using a standard inertial graph partitioning algorithm") -- input
preparation shared by both sides of every parity check, checked on CPU."""
from __future__ import annotations

import numpy as np

from datagen import gen_config_points
from datagen.partition import inertial_order


def test_is_a_deterministic_permutation():
    X, _ = gen_config_points("C4", 0, 0.0005)
    p = inertial_order(X, device="cpu")
    assert np.array_equal(np.sort(p), np.arange(len(X)))
    assert np.array_equal(p, inertial_order(X, device="cpu"))


def test_first_cut_is_the_principal_axis_median():
    # an elongated cloud rotated by 30 degrees: the inertial axis is the long
    # one, and the first bisection splits at the median of the projections on it
    rng = np.random.default_rng(3)
    n = 4096
    Y = rng.standard_normal((n, 2)) * np.array([10.0, 1.0])
    t = np.pi / 6
    R = np.array([[np.cos(t), -np.sin(t)], [np.sin(t), np.cos(t)]])
    X = (Y @ R.T).astype(np.float32)
    p = inertial_order(X, device="cpu", align=1024)
    proj = Y[:, 0]  # coordinate along the principal axis
    first, second = proj[p[: n // 2]], proj[p[n // 2:]]
    assert first.max() <= second.min() or second.max() <= first.min()


def test_order_is_local_and_blocks_are_compact():
    X, truth = gen_config_points("C4", 0, 0.003)  # 192,000 points on 10 unit spheres
    p = inertial_order(X, device="cpu", align=1024)
    Y, ty = X[p], truth[p]
    step = np.linalg.norm(np.diff(Y, axis=0), axis=1)
    assert np.median(step) < 0.1 * np.median(np.linalg.norm(np.diff(X, axis=0), axis=1))
    # 1,024-id blocks (1/19 of a sphere): almost all lie on one sphere, in a cap
    # (generation order: every block spans its whole sphere, extent ~2)
    nb = len(Y) // 1024
    one = [len(np.unique(ty[b * 1024:(b + 1) * 1024])) == 1 for b in range(nb)]
    ext = [float(np.max(Y[b * 1024:(b + 1) * 1024].max(0) - Y[b * 1024:(b + 1) * 1024].min(0)))
           for b in range(nb)]
    assert sum(one) >= 0.9 * nb
    assert np.median([e for e, o in zip(ext, one) if o]) < 1.25


def test_degenerate_inputs():
    assert np.array_equal(inertial_order(np.zeros((1, 3), np.float32), device="cpu"), [0])
    dup = np.zeros((300, 2), np.float32)  # all points equal: zero covariance, order kept
    assert np.array_equal(inertial_order(dup, device="cpu"), np.arange(300))
