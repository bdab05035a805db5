"""Point-set generators for configs C1..C5 (BASELINE.json ``configs``).

Conventions (SURVEY.md §8(d) "Synthetic inputs"):
  * numpy ``default_rng(seed)`` (PCG64); every draw in fp64, in the order the
    recipe lists, cast to fp32 at the end;
  * points stay in generation order (cluster-major, noise last), no spatial sort;
  * seed 0 unless stated.
Each generator returns ``(X float32 [N, d], truth int32 [N])`` where ``truth``
is the generating component (-1 for the uniform noise of C1); ``truth`` is
only used for reporting, never by either side of the parity check.
"""
from __future__ import annotations

import numpy as np

# name -> (N, d, k, M, eps_factor)   (BASELINE.json configs[0..4])
CONFIGS = {
    "C1": dict(N=10_000, d=2, k=16, M=8, eps_factor=1.5),
    "C2": dict(N=2_000_000, d=50, k=32, M=16, eps_factor=1.2),
    "C3": dict(N=4_000_000, d=10, k=100, M=50, eps_factor=1.5),
    "C4": dict(N=64_000_000, d=3, k=100, M=50, eps_factor=1.5),
    "C5": dict(N=256_000_000, d=5, k=100, M=50, eps_factor=1.5),
}


def _unit_sphere(rng: np.random.Generator, n: int, d: int) -> np.ndarray:
    """n points uniform on the unit (d-1)-sphere: normalised Gaussians (fp64)."""
    g = rng.standard_normal((n, d))
    nrm = np.sqrt(np.einsum("ij,ij->i", g, g))
    # a zero-norm Gaussian draw has probability 0; guard anyway
    nrm[nrm == 0.0] = 1.0
    return g / nrm[:, None]


def gen_c1(seed: int = 0, n_per_blob: int = 2375, n_noise: int = 500):
    """C1: 4 isotropic Gaussian blobs, sigma 0.05, centres (cos t, sin t) for
    t = 0, pi/2, pi, 3pi/2, drawn blob by blob; then uniform noise in
    [-1.5, 1.5]^2 (BASELINE.json configs[0])."""
    rng = np.random.default_rng(seed)
    parts, truth = [], []
    for b in range(4):
        t = b * np.pi / 2.0
        c = np.array([np.cos(t), np.sin(t)])
        parts.append(c + 0.05 * rng.standard_normal((n_per_blob, 2)))
        truth.append(np.full(n_per_blob, b, np.int32))
    parts.append(rng.uniform(-1.5, 1.5, size=(n_noise, 2)))
    truth.append(np.full(n_noise, -1, np.int32))
    return np.concatenate(parts).astype(np.float32), np.concatenate(truth)


def gen_c2(seed: int = 0, n_per: int = 200_000, d: int = 50, n_centres: int = 10):
    """C2: 10-component Gaussian mixture in 50-D, centres ~ N(0, 0.04 I)
    (i.e. 0.2 * N(0, I)), per-cluster sigma 0.01, equal weights
    (BASELINE.json configs[1])."""
    rng = np.random.default_rng(seed)
    centres = 0.2 * rng.standard_normal((n_centres, d))
    parts, truth = [], []
    for c in range(n_centres):
        parts.append(centres[c] + 0.01 * rng.standard_normal((n_per, d)))
        truth.append(np.full(n_per, c, np.int32))
    return np.concatenate(parts).astype(np.float32), np.concatenate(truth)


def gen_c3(seed: int = 0, n_inner: int = 1_000_000, n_outer: int = 3_000_000, d: int = 10):
    """C3 (= the paper's Uniform2S): n_inner points uniform on the
    origin-centred sphere surface of radius 0.1, then n_outer on radius 1.0."""
    rng = np.random.default_rng(seed)
    inner = 0.1 * _unit_sphere(rng, n_inner, d)
    outer = 1.0 * _unit_sphere(rng, n_outer, d)
    X = np.concatenate([inner, outer]).astype(np.float32)
    truth = np.concatenate([np.zeros(n_inner, np.int32), np.ones(n_outer, np.int32)])
    return X, truth


def _sphere_clusters(seed: int, d: int, n_per: int, n_centres: int = 10,
                     box: float = 20.0, min_sep: float = 3.0):
    rng = np.random.default_rng(seed)
    centres = []
    while len(centres) < n_centres:  # sequential rejection
        c = rng.uniform(-box, box, size=d)
        if all(np.sqrt(np.sum((c - e) ** 2)) >= min_sep for e in centres):
            centres.append(c)
    X = np.empty((n_centres * n_per, d), np.float32)
    truth = np.empty(n_centres * n_per, np.int32)
    for i, c in enumerate(centres):
        X[i * n_per:(i + 1) * n_per] = (c + _unit_sphere(rng, n_per, d)).astype(np.float32)
        truth[i * n_per:(i + 1) * n_per] = i
    return X, truth


def gen_c4(seed: int = 0, n_per: int = 6_400_000):
    """C4: 10 equal clusters uniform on unit 2-sphere surfaces, centres uniform in
    [-20, 20]^3 with rejection below separation 3 (BASELINE.json configs[3])."""
    return _sphere_clusters(seed, 3, n_per)


def gen_c5(seed: int = 0, n_per: int = 25_600_000):
    """C5: as C4 with d = 5 (unit 4-spheres) (BASELINE.json configs[4])."""
    return _sphere_clusters(seed, 5, n_per)


def gen_config_points(name: str, seed: int = 0, scale: float = 1.0):
    """Points of config ``name``; ``scale`` < 1 shrinks every cluster
    proportionally (same recipe, fewer points) for tests."""
    s = lambda n: max(1, int(round(n * scale)))
    if name == "C1":
        return gen_c1(seed, s(2375), s(500))
    if name == "C2":
        return gen_c2(seed, s(200_000))
    if name == "C3":
        return gen_c3(seed, s(1_000_000), s(3_000_000))
    if name == "C4":
        return gen_c4(seed, s(6_400_000))
    if name == "C5":
        return gen_c5(seed, s(25_600_000))
    raise KeyError(name)
