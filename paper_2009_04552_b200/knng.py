"""Binding of libknng.so (C-ABI: include/knng.h) -- the exact kNN-graph
builder: the stage before the clustering stage
("constructing k-NNG is the dominant cost"; Table 2, PAPER.md:21-36,
times GOFMM's approximate builder).  Two exact GPU builders: a uniform-grid
cell search for d <= 5 and a certified brute force (fp32 candidate heaps,
fp64 re-rank) for d <= 64.  Rows exclude self and are ordered by (fp64
distance, index), the graph convention of include/kdb.h.  It is timed
separately from the clustering stage (north_star: the graph is input) --
`bench.py --stage knng`.  Argument marshalling only; no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KNNG_LIBRARY") or os.path.join(_HERE, "lib", "libknng.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built (run make)")
        L = C.CDLL(LIB_PATH)
        L.knng_grid_ws.argtypes = [C.c_int64]
        L.knng_grid_ws.restype = C.c_size_t
        L.knng_ladder.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int, C.c_float, C.c_void_p,
                                  C.c_void_p]
        L.knng_grid.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_double,
                                C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                C.POINTER(C.c_int64)]
        L.knng_grid_rows.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_double,
                                     C.c_double, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_size_t, C.c_void_p, C.POINTER(C.c_int64)]
        L.knng_brute.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.knng_exact_row.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def estimate_radius(Xd: torch.Tensor, k: int, n_samples: int = 256, quantile: float = 0.99) -> float:
    """Upper estimate of the k-th-neighbour radius from a log-ladder histogram of
    the distances of ``n_samples`` evenly spaced sample points to all points."""
    n, d = Xd.shape
    lo = Xd.min(0).values.double(); hi = Xd.max(0).values.double()
    diag = float(torch.sqrt(((hi - lo) ** 2).sum()).item()) or 1.0
    r_lo = diag * 2.0 ** -16
    S = min(n_samples, n)
    samples = torch.linspace(0, n - 1, S, device=Xd.device).round().to(torch.int32)
    hist = torch.zeros(S * 64, dtype=torch.int32, device=Xd.device)
    st = torch.cuda.current_stream().cuda_stream
    if _load().knng_ladder(Xd.data_ptr(), n, d, samples.data_ptr(), S, r_lo, hist.data_ptr(), st):
        raise RuntimeError("knng_ladder failed")
    cum = hist.view(S, 64).cumsum(1).cpu().numpy()
    b = np.argmax(cum >= k + 1, axis=1)              # first bucket reaching k+1 (self included)
    r_up = r_lo * 2.0 ** ((b + 1) / 4.0)
    return float(np.quantile(r_up, quantile))


def build_knng_grid(X, k: int, h: float | None = None, device: str = "cuda", rows=None):
    """Exact self-excluded kNN graph of X (np/torch float32 [n, d], d <= 5).
    Returns (nbr int32 [n,k], dist float32 [n,k], info dict) as CUDA tensors.
    rows=(begin, end): only query rows [begin, end) (one rank's rows; every
    point stays a candidate) -> [end - begin, k] tensors (knng_grid_rows)."""
    Xd = torch.as_tensor(np.ascontiguousarray(X, np.float32) if isinstance(X, np.ndarray) else X)
    Xd = Xd.to(device=device, dtype=torch.float32).contiguous()
    n, d = Xd.shape
    if not (1 <= d <= 5) or not (1 <= k <= n - 1):
        raise ValueError("need d <= 5 and 1 <= k <= n-1")
    if h is None:
        h = 1.05 * estimate_radius(Xd, k)
    lo = (Xd.min(0).values.double() - 2.0 * h).cpu().numpy().astype(np.float64)
    hi = Xd.max(0).values.double().cpu().numpy()
    bits = min(63 // d, 21)
    span = float(np.max((hi - lo) / h)) + 2
    if span >= (1 << bits) - 2:
        h = (np.max(hi - lo) + 4 * h) / ((1 << bits) - 4)  # coarsen: exact either way
        lo = (Xd.min(0).values.double() - 2.0 * h).cpu().numpy().astype(np.float64)
    qb, qe = (0, n) if rows is None else (int(rows[0]), int(rows[1]))
    if not 0 <= qb <= qe <= n:
        raise ValueError("rows must satisfy 0 <= begin <= end <= n")
    nbr = torch.empty((qe - qb, k), dtype=torch.int32, device=device)
    dist = torch.empty((qe - qb, k), dtype=torch.float32, device=device)
    L = _load()
    ws_bytes = L.knng_grid_ws(n)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=device)
    lo_c = (C.c_double * 8)(*lo.tolist())
    nfb = C.c_int64(0)
    st = torch.cuda.current_stream().cuda_stream
    span = float(np.max((hi - lo) / h)) + 2
    diag = float(np.sqrt(np.sum((hi - lo) ** 2)))
    rc = L.knng_grid_rows(Xd.data_ptr(), n, d, k, float(h), lo_c, span, diag, qb, qe - qb, nbr.data_ptr(),
                          dist.data_ptr(), ws.data_ptr(), ws_bytes, st, C.byref(nfb))
    if rc:
        raise RuntimeError(f"knng_grid failed rc={rc}")
    del ws
    return nbr, dist, dict(h=float(h), n_fallback=int(nfb.value))


def build_knng_brute(X, k: int, margin: int = 32, device: str = "cuda"):
    """Exact self-excluded kNN graph of X (float32 [n, d], any d <= 64) by GPU
    brute force: fp32 candidate heaps of size k + margin, exact fp64 re-rank by
    (distance, index), certificate-checked; failing rows are recomputed over all
    points.  Same rows as ``knn_cpu.knn_bruteforce``.  Returns CUDA tensors
    (nbr int32 [n,k], dist float32 [n,k], info dict)."""
    Xd = torch.as_tensor(np.ascontiguousarray(X, np.float32) if isinstance(X, np.ndarray) else X)
    Xd = Xd.to(device=device, dtype=torch.float32).contiguous()
    n, d = Xd.shape
    if not (1 <= d <= 64) or not (1 <= k <= n - 1):
        raise ValueError("need d <= 64 and 1 <= k <= n-1")
    Kp = min(n - 1, k + margin, 256)
    L = _load()
    hs = torch.empty(n * Kp, dtype=torch.float32, device=device)
    hi = torch.empty(n * Kp, dtype=torch.int32, device=device)
    hc = torch.empty(n, dtype=torch.int32, device=device)
    nbr = torch.empty((n, k), dtype=torch.int32, device=device)
    dist = torch.empty((n, k), dtype=torch.float32, device=device)
    fail = torch.empty(n, dtype=torch.int32, device=device)
    nfail = torch.zeros(1, dtype=torch.int32, device=device)
    st = torch.cuda.current_stream().cuda_stream
    rc = L.knng_brute(Xd.data_ptr(), n, d, k, Kp, hs.data_ptr(), hi.data_ptr(), hc.data_ptr(), nbr.data_ptr(),
                      dist.data_ptr(), fail.data_ptr(), nfail.data_ptr(), st)
    if rc:
        raise RuntimeError(f"knng_brute failed rc={rc}")
    del hs, hi, hc
    nf = int(nfail.item())
    if nf:
        rows = fail[:nf].cpu().tolist()
        buf = torch.empty(n, dtype=torch.float64, device=device)
        for q in rows:
            if L.knng_exact_row(Xd.data_ptr(), n, d, int(q), buf.data_ptr(), st):
                raise RuntimeError("knng_exact_row failed")
            order = torch.sort(buf, stable=True).indices[:k]   # stable: ties by ascending index
            nbr[q] = order.to(torch.int32)
            dist[q] = buf[order].to(torch.float32)
    return nbr, dist, dict(candidates=Kp, certificate_failures=nf)
