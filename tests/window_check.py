"""Full-size oracle parity by exact cluster windows (test infrastructure).

C4 and C5 place 10 clusters on unit spheres whose centres are >= 3 apart
(datagen/points.py ``_sphere_clusters``), so points of different clusters are
>= 1 apart while every kNN radius is < 0.1: no kNN entry crosses a cluster.
The rows of one cluster therefore form a CLOSED exact kNN graph (every id in
the window lies in the window; this module checks it on the device before
using it).  In generation order a cluster is an id range [s, e); in the
inertial order of PAPER.md:45 (datagen/partition.py) it is a set of ids, and
the window maps them to 0..n-1 in increasing order -- a monotone map, so
minimum ids (canonical labels), a < b and the (a, b) order of the MSF are
kept.  The exact outputs decompose:

  * core flags and border labels are row-local (Alg. 1 l.3-8, Lemma 1(ii));
  * the candidate edges of a window join window vertices only, so the MSF of
    the whole graph is the disjoint union of the windows' MSFs (Kruskal under a
    strict order restricted to a union of components, Thm. 2);
  * a canonical label (minimum core id of the component) is a window id.

So the whole-workload oracle result is the union of per-window oracle runs with
ids shifted by s, and the GPU result of the FULL benchmarked run restricted to a
window must equal its window's oracle result element by element.

Only tests/ and tools/window_parity.py use this module; it calls the oracle
(oracle/) on the host and reads GPU outputs as plain tensors.
"""
from __future__ import annotations

import hashlib
import threading
import time

import numpy as np
import torch

import oracle


def cluster_windows(truth: np.ndarray):
    """One window per generator cluster, in cluster-id order: (s, e) when the
    cluster's ids are one contiguous range (generation order: cluster-major),
    else the sorted member ids (int64 array) -- the inertial order of
    PAPER.md:45 (datagen/partition.py) interleaves clusters in id space."""
    t = np.asarray(truth)
    cuts = np.flatnonzero(t[1:] != t[:-1]) + 1
    b = np.concatenate([[0], cuts, [len(t)]])
    runs = [(int(b[i]), int(b[i + 1])) for i in range(len(b) - 1)]
    if len({int(t[s]) for s, _ in runs}) == len(runs):  # every cluster is one run
        return sorted(runs, key=lambda r: int(t[r[0]]))
    order = np.argsort(t, kind="stable")
    ids, first, counts = np.unique(t[order], return_index=True, return_counts=True)
    return [np.ascontiguousarray(order[f:f + c], np.int64) for f, c in zip(first, counts)]


def is_range(win) -> bool:
    return isinstance(win, tuple)


def win_size(win) -> int:
    return win[1] - win[0] if is_range(win) else len(win)


def _local(J: torch.Tensor, win, m_dev=None) -> torch.Tensor:
    """Global ids -> window-local ids (monotone: order and minima are kept);
    padding (-1) stays -1.  Ids outside the window map to garbage (callers
    check closure first)."""
    if is_range(win):
        return torch.where(J >= 0, J - win[0], J)
    loc = torch.searchsorted(m_dev, J.contiguous())
    return torch.where(J >= 0, loc, J)


def _rows(x: torch.Tensor, win, a: int, b: int, m_dev=None) -> torch.Tensor:
    """Window rows [a, b) (window-local row positions) of a [N, k] device tensor."""
    if is_range(win):
        return x[win[0] + a:win[0] + b]
    return x[m_dev[a:b]]


def _mdev(win, device):
    return None if is_range(win) else torch.from_numpy(win).to(device)


def window_closed(nbr: torch.Tensor, win, e=None, chunk: int = 1 << 22) -> bool:
    """Every id stored in the window's rows is padding (-1) or a window id."""
    if e is not None:
        win = (win, e)
    n = win_size(win)
    if is_range(win):
        s, e = win
        for a in range(s, e, chunk):
            J = nbr[a:min(a + chunk, e)]
            if not bool(((J == -1) | ((J >= s) & (J < e))).all()):
                return False
        return True
    m = _mdev(win, nbr.device)
    member = torch.zeros(nbr.shape[0], dtype=torch.bool, device=nbr.device)
    member[m] = True
    for a in range(0, n, chunk):
        J = _rows(nbr, win, a, min(a + chunk, n), m).long()
        ok = (J == -1) | ((J >= 0) & (J < nbr.shape[0]) & member[J.clamp(0, nbr.shape[0] - 1)])
        if not bool(ok.all()):
            return False
    return True


def input_checksum(nbr: torch.Tensor, dist: torch.Tensor, win, e=None, chunk: int = 1 << 21) -> str:
    """Position-weighted int64 checksum of the window's rows with ids mapped to
    window-local ids (the bytes the oracle sees), computed on the device: a
    cache key for the stored oracle digests, not a cryptographic hash."""
    if e is not None:
        win = (win, e)
    k = nbr.shape[1]
    n = win_size(win)
    m = _mdev(win, nbr.device)
    acc = torch.zeros((), dtype=torch.int64, device=nbr.device)
    col = torch.arange(1, k + 1, dtype=torch.int64, device=nbr.device)
    for a in range(0, n, chunk):
        b = min(a + chunk, n)
        J = _local(_rows(nbr, win, a, b, m).long(), win, m)
        W = _rows(dist, win, a, b, m).contiguous().view(torch.int32).long()
        row = torch.arange(a + 1, b + 1, dtype=torch.int64, device=nbr.device)[:, None]
        x = (J * 1000003 + W) * (row * 7919 + col * 104729)
        acc += x.sum()
    return f"{int(acc.item()) & ((1 << 64) - 1):016x}"


def digest(core, labels, msf_a, msf_b, msf_w) -> str:
    """sha256 over window-local outputs (weights compared without the sign bit,
    the parity rule's -0 == +0)."""
    h = hashlib.sha256()
    for x, dt in ((core, np.uint8), (labels, np.int32), (msf_a, np.uint32), (msf_b, np.uint32)):
        h.update(np.ascontiguousarray(x, dt).tobytes())
    h.update((np.ascontiguousarray(msf_w, np.float32).view(np.uint32) & np.uint32(0x7fffffff)).tobytes())
    return h.hexdigest()


def gpu_window(full: dict, win, e=None) -> dict:
    """The full-graph GPU outputs restricted to a window, ids mapped to
    window-local ones (full: core uint8[N], comp/labels int32[N], MSF a/b/w
    sorted by (a, b))."""
    if e is not None:
        win = (win, e)
    a, b = full["msf_a"], full["msf_b"]
    if is_range(win):
        s, e = win
        lo, hi = np.searchsorted(a, s, "left"), np.searchsorted(a, e, "left")
        sel = slice(lo, hi)
        loc = lambda x: np.where(x >= 0, x - s, x)
        rows = slice(s, e)
        inside = lambda x: (x >= s) & (x < e)
        span = (int(lo), int(hi))
    else:
        m = win
        mask = np.zeros(len(full["core"]), bool)
        mask[m] = True
        inside = lambda x: mask[np.clip(x, 0, len(mask) - 1)] & (x >= 0) & (x < len(mask))
        sel = np.flatnonzero(inside(a.astype(np.int64)))
        loc = lambda x: np.where(x >= 0, np.searchsorted(m, x), x)
        rows = m
        span = (0, int(len(sel)))
    lab = full["labels"][rows].astype(np.int64)
    comp = full["comp"][rows].astype(np.int64)
    wa, wb = a[sel].astype(np.int64), b[sel].astype(np.int64)
    out = dict(core=full["core"][rows], labels=loc(lab).astype(np.int32), comp=loc(comp).astype(np.int32),
               msf_a=loc(wa).astype(np.uint32), msf_b=loc(wb).astype(np.uint32), msf_w=full["msf_w"][sel])
    # every MSF edge of the window joins window vertices
    out["edges_inside"] = bool(np.all(inside(wb)))
    # fp64 weight of the window's forest in O1 key order (the oracle's summation order)
    w = out["msf_w"]
    order = np.lexsort((out["msf_b"], out["msf_a"], w.view(np.uint32) & np.uint32(0x7fffffff)))
    out["msf_weight"] = float(np.sum(w[order].astype(np.float64))) if len(w) else 0.0
    out["span"] = span
    return out


def window_graph_host(nbr: torch.Tensor, dist: torch.Tensor, win, e=None):
    """The window's rows on the host with ids mapped to window-local ones (the oracle's input)."""
    if e is not None:
        win = (win, e)
    m = _mdev(win, nbr.device)
    n = win_size(win)
    J = _local(_rows(nbr, win, 0, n, m).long(), win, m).to(torch.int32).cpu().numpy()
    return np.ascontiguousarray(J, np.int32), np.ascontiguousarray(_rows(dist, win, 0, n, m).cpu().numpy(), np.float32)


def run_oracle(nbr_w: np.ndarray, dist_w: np.ndarray, M: int, eps: float) -> dict:
    """The oracle (single-threaded C++) on one window; adds wall seconds."""
    t = time.perf_counter()
    r = oracle.kdbscan(nbr_w, dist_w, M, np.float32(eps))
    r["wall_s"] = time.perf_counter() - t
    r["digest"] = digest(r["core"], r["labels"], r["msf_a"], r["msf_b"], r["msf_w"])
    return r


def compare(got: dict, exp: dict, rel_tol: float = 1e-6) -> list:
    """Element-by-element parity of one window; returns the failures (empty = pass)."""
    bad = []
    if not np.array_equal(got["core"], exp["core"]):
        bad.append("core")
    core = exp["core"].astype(bool)
    if not np.array_equal(got["comp"][core], exp["labels"][core]) or not np.all(got["comp"][~core] == -1):
        bad.append("comp")
    if not np.array_equal(got["labels"], exp["labels"]):
        bad.append("labels")
    if not got["edges_inside"]:
        bad.append("msf edge leaves the window")
    if len(got["msf_a"]) != len(exp["msf_a"]) or not (np.array_equal(got["msf_a"], exp["msf_a"]) and
                                                     np.array_equal(got["msf_b"], exp["msf_b"])):
        bad.append("msf edge set")
    elif not np.array_equal(got["msf_w"].view(np.uint32) & 0x7fffffff, exp["msf_w"].view(np.uint32) & 0x7fffffff):
        bad.append("msf weights")
    ew = exp["msf_weight"]
    if abs(got["msf_weight"] - ew) > rel_tol * max(abs(ew), 1e-300):
        bad.append(f"msf weight {got['msf_weight']!r} vs {ew!r}")
    return bad


class MemGate:
    """Admit oracle windows while the host has room (each needs ~36 B per entry)."""

    def __init__(self, need_bytes: int, workers: int):
        self.need, self.sem = need_bytes, threading.Semaphore(max(1, workers))

    @staticmethod
    def available() -> int:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
        return 0
