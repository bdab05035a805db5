"""CPU oracle for the kNN-DBSCAN clustering stage -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path never does.  The arithmetic lives in ``kdb_oracle.cpp`` (plain
C++17, see its header for the passages each step follows); this module only
marshals numpy arrays through ctypes.

Parity status: every function here is pinned by tests/test_oracle_pins.py
(no "parity unpinned" entries).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build() -> str:
    """Compile liboracle.so (plain g++; building the checker is not using it)."""
    src = os.path.join(_HERE, "kdb_oracle.cpp")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", _LIB_PATH, src])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        i64, i32, f32 = C.c_int64, C.c_int32, C.c_float
        lib.oracle_core_mark.argtypes = [i64, i32, P, i32, f32, P]
        lib.oracle_candidate_count.argtypes = [i64, i32, P, P, P, f32, i32]
        lib.oracle_candidate_count.restype = i64
        lib.oracle_candidates.argtypes = [i64, i32, P, P, P, f32, i32, P, P, P, i64]
        lib.oracle_candidates.restype = i64
        lib.oracle_kruskal.argtypes = [i64, i64, P, P, P, P, P, P, P, P, i64, P, P]
        lib.oracle_border.argtypes = [i64, i32, P, P, P, f32, P, P]
        lib.oracle_kdbscan.argtypes = [i64, i32, P, P, i32, f32, i32, P, P, P, P, P, i64, P, P, P]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _graph(nbr, dist):
    nbr = np.ascontiguousarray(nbr, np.int32)
    dist = np.ascontiguousarray(dist, np.float32)
    if nbr.shape != dist.shape or nbr.ndim != 2:
        raise ValueError("nbr/dist must be [n, k] arrays of equal shape")
    return nbr, dist


def core_mark(dist, M: int, eps) -> np.ndarray:
    dist = np.ascontiguousarray(dist, np.float32)
    n, k = dist.shape
    core = np.zeros(n, np.uint8)
    if _load().oracle_core_mark(n, k, _p(dist), M, np.float32(eps), _p(core)):
        raise ValueError("bad arguments")
    return core


def _cols(edge_cols, k):
    c = k if edge_cols is None else int(edge_cols)
    if not 1 <= c <= k:
        raise ValueError(f"edge_cols must be in [1, k={k}]")
    return c


def candidates(nbr, dist, core, eps, edge_cols=None):
    """Candidate multiset (a, b, w) in row order, from
    the first `edge_cols` columns (default all k; edge_cols = M is Def. 6)."""
    nbr, dist = _graph(nbr, dist)
    core = np.ascontiguousarray(core, np.uint8)
    n, k = nbr.shape
    kc = _cols(edge_cols, k)
    lib = _load()
    m = lib.oracle_candidate_count(n, k, _p(nbr), _p(dist), _p(core), np.float32(eps), kc)
    a = np.empty(m, np.uint32); b = np.empty(m, np.uint32); w = np.empty(m, np.float32)
    lib.oracle_candidates(n, k, _p(nbr), _p(dist), _p(core), np.float32(eps), kc, _p(a), _p(b), _p(w), m)
    return a, b, w


def kruskal(n: int, a, b, w, is_vertex):
    """Kruskal MSF under key (mono(w), min id, max id) on an explicit multigraph."""
    a = np.ascontiguousarray(a, np.uint32); b = np.ascontiguousarray(b, np.uint32)
    w = np.ascontiguousarray(w, np.float32)
    is_vertex = np.ascontiguousarray(is_vertex, np.uint8)
    comp = np.empty(n, np.int32)
    cap = max(n - 1, 0)
    ma = np.empty(cap, np.uint32); mb = np.empty(cap, np.uint32); mw = np.empty(cap, np.float32)
    cnt = C.c_int64(0); tot = C.c_double(0.0)
    rc = _load().oracle_kruskal(n, len(a), _p(a), _p(b), _p(w), _p(is_vertex), _p(comp),
                                _p(ma), _p(mb), _p(mw), cap, C.byref(cnt), C.byref(tot))
    if rc:
        raise RuntimeError(f"oracle_kruskal rc={rc}")
    c = cnt.value
    return comp, ma[:c].copy(), mb[:c].copy(), mw[:c].copy(), tot.value


def border(nbr, dist, core, eps, comp):
    nbr, dist = _graph(nbr, dist)
    n, k = nbr.shape
    core = np.ascontiguousarray(core, np.uint8)
    comp = np.ascontiguousarray(comp, np.int32)
    labels = np.empty(n, np.int32)
    _load().oracle_border(n, k, _p(nbr), _p(dist), _p(core), np.float32(eps), _p(comp), _p(labels))
    return labels


def kdbscan(nbr, dist, M: int, eps, edge_cols=None):
    """The whole clustering stage (Alg. 1 as its plain definition).

    edge_cols: candidate edges come from the first edge_cols columns of each
    row (default k = reading #3; edge_cols = M is the paper's direct
    M-reachability, Def. 6 PAPER.md:958-962 / Thm. 2(ii)).

    Returns dict(core uint8[n], labels int32[n], msf_a/msf_b uint32[c] sorted by
    (a, b), msf_w float32[c], msf_weight float (fp64 sum in key order),
    times [core, msf, border] seconds).
    """
    nbr, dist = _graph(nbr, dist)
    n, k = nbr.shape
    kc = _cols(edge_cols, k)
    core = np.empty(n, np.uint8)
    labels = np.empty(n, np.int32)
    cap = max(n - 1, 0)
    ma = np.empty(cap, np.uint32); mb = np.empty(cap, np.uint32); mw = np.empty(cap, np.float32)
    cnt = C.c_int64(0); tot = C.c_double(0.0)
    times = np.zeros(3, np.float64)
    rc = _load().oracle_kdbscan(n, k, _p(nbr), _p(dist), int(M), np.float32(eps), kc, _p(core),
                                _p(labels), _p(ma), _p(mb), _p(mw), cap, C.byref(cnt),
                                C.byref(tot), _p(times))
    if rc == -1:
        raise ValueError("bad arguments (M, k or eps)")
    if rc:
        raise RuntimeError(f"oracle_kdbscan rc={rc}")
    c = cnt.value
    return dict(core=core, labels=labels, msf_a=ma[:c].copy(), msf_b=mb[:c].copy(),
                msf_w=mw[:c].copy(), msf_weight=tot.value, times=times)
