"""Full-size oracle parity by exact cluster windows (test infrastructure).

C4 and C5 place 10 clusters on unit spheres whose centres are >= 3 apart
(datagen/points.py ``_sphere_clusters``), so points of different clusters are
>= 1 apart while every kNN radius is < 0.1: no kNN entry crosses a cluster,
and ids are cluster-major.  Rows [s, e) of one cluster therefore form a CLOSED
exact kNN graph (every id in the window lies in the window; this module checks
it on the device before using it), and the exact outputs decompose:

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
    """[(s, e)] contiguous ranges of equal generator cluster id (cluster-major)."""
    t = np.asarray(truth)
    cuts = np.flatnonzero(t[1:] != t[:-1]) + 1
    b = np.concatenate([[0], cuts, [len(t)]])
    return [(int(b[i]), int(b[i + 1])) for i in range(len(b) - 1)]


def window_closed(nbr: torch.Tensor, s: int, e: int, chunk: int = 1 << 22) -> bool:
    """Every id stored in rows [s, e) is padding (-1) or lies in [s, e)."""
    for a in range(s, e, chunk):
        J = nbr[a:min(a + chunk, e)]
        if not bool(((J == -1) | ((J >= s) & (J < e))).all()):
            return False
    return True


def input_checksum(nbr: torch.Tensor, dist: torch.Tensor, s: int, e: int, chunk: int = 1 << 21) -> str:
    """Position-weighted int64 checksum of rows [s, e) with ids shifted by -s
    (the bytes the oracle sees), computed on the device: a cache key for the
    stored oracle digests, not a cryptographic hash."""
    k = nbr.shape[1]
    acc = torch.zeros((), dtype=torch.int64, device=nbr.device)
    col = torch.arange(1, k + 1, dtype=torch.int64, device=nbr.device)
    for a in range(s, e, chunk):
        b = min(a + chunk, e)
        J = nbr[a:b].long()
        J = torch.where(J >= 0, J - s, J)
        W = dist[a:b].contiguous().view(torch.int32).long()
        row = torch.arange(a - s + 1, b - s + 1, dtype=torch.int64, device=nbr.device)[:, None]
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


def gpu_window(full: dict, s: int, e: int) -> dict:
    """The full-graph GPU outputs restricted to window [s, e), ids shifted to
    window-local (full: core uint8[N], comp/labels int32[N], sorted MSF a/b/w)."""
    a, b = full["msf_a"], full["msf_b"]
    lo, hi = np.searchsorted(a, s, "left"), np.searchsorted(a, e, "left")
    lab = full["labels"][s:e].astype(np.int64)
    comp = full["comp"][s:e].astype(np.int64)
    out = dict(core=full["core"][s:e], labels=np.where(lab >= 0, lab - s, lab).astype(np.int32),
               comp=np.where(comp >= 0, comp - s, comp).astype(np.int32),
               msf_a=(a[lo:hi].astype(np.int64) - s).astype(np.uint32),
               msf_b=(b[lo:hi].astype(np.int64) - s).astype(np.uint32), msf_w=full["msf_w"][lo:hi])
    # every MSF edge of the window joins window vertices
    out["edges_inside"] = bool(np.all((b[lo:hi] >= s) & (b[lo:hi] < e)))
    # fp64 weight of the window's forest in O1 key order (the oracle's summation order)
    w = out["msf_w"]
    order = np.lexsort((out["msf_b"], out["msf_a"], w.view(np.uint32) & np.uint32(0x7fffffff)))
    out["msf_weight"] = float(np.sum(w[order].astype(np.float64))) if len(w) else 0.0
    out["span"] = (int(lo), int(hi))
    return out


def window_graph_host(nbr: torch.Tensor, dist: torch.Tensor, s: int, e: int):
    """Rows [s, e) on the host with ids shifted to window-local (the oracle's input)."""
    J = nbr[s:e]
    J = torch.where(J >= 0, J - s, J).cpu().numpy()
    return np.ascontiguousarray(J, np.int32), np.ascontiguousarray(dist[s:e].cpu().numpy(), np.float32)


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
