"""fp64 brute-force k-NN rows on the GPU with plain torch ops (test
infrastructure): the independent spot check of the kNN-graph builder on
sampled rows of full-size graphs (north_star: "spot-checked against brute
force on sampled rows").

Same definition as datagen/knn_cpu.py, written with elementwise torch ops so
every operation rounds like the CPU version: fp32 coordinates promoted to
fp64, acc = ((0 + d_0^2) + d_1^2) + ... in dimension order (separate multiply
and add kernels: no fused multiply-add), sqrt; self excluded; rows ordered by
(distance, index); stored as fp32 / int32.
"""
from __future__ import annotations

import torch


def knn_rows_torch(X: torch.Tensor, rows: torch.Tensor, k: int, q_batch: int = 256, p_chunk: int = 1 << 22,
                   cand=None):
    """Exact self-excluded kNN rows of query ids ``rows`` against all of X
    (device float32 [n, d]), or against the ids [cand[0], cand[1]) when the
    caller has proved no other point can be among the k nearest (see
    separated_clusters).  Returns (nbr int32 [m, k], dist float32 [m, k])."""
    lo, hi = (0, X.shape[0]) if cand is None else cand
    n, d = hi, X.shape[1]
    m = rows.numel()
    out_n = torch.empty((m, k), dtype=torch.int32, device=X.device)
    out_d = torch.empty((m, k), dtype=torch.float32, device=X.device)
    extra = 8  # candidates kept per chunk beyond k: ties at the cut are re-ranked exactly below
    for q0 in range(0, m, q_batch):
        qi = rows[q0:q0 + q_batch].long()
        Q = X[qi].double()
        best_d, best_i = None, None
        for p0 in range(lo, n, p_chunk):
            P = X[p0:min(p0 + p_chunk, n)].double()
            acc = torch.zeros((Q.shape[0], P.shape[0]), dtype=torch.float64, device=X.device)
            for t in range(d):
                df = Q[:, t:t + 1] - P[None, :, t]
                acc = acc + df * df
            dd = torch.sqrt(acc)
            ids = torch.arange(p0, p0 + P.shape[0], device=X.device)
            dd[ids[None, :] == qi[:, None]] = float("inf")  # exclude self
            kk = min(k + extra, P.shape[0])
            v, j = torch.topk(dd, kk, dim=1, largest=False)
            j = j + p0
            best_d = v if best_d is None else torch.cat([best_d, v], 1)
            best_i = j if best_i is None else torch.cat([best_i, j], 1)
            if best_d.shape[1] > 4 * (k + extra):  # keep the merged candidate lists short
                v, sel = torch.topk(best_d, k + extra, dim=1, largest=False)
                best_d, best_i = v, torch.gather(best_i, 1, sel)
        # exact order by (distance, index): sort by index, then stable by distance
        o = torch.argsort(best_i, dim=1)
        best_d, best_i = torch.gather(best_d, 1, o), torch.gather(best_i, 1, o)
        o = torch.sort(best_d, dim=1, stable=True).indices
        best_d, best_i = torch.gather(best_d, 1, o)[:, :k], torch.gather(best_i, 1, o)[:, :k]
        out_n[q0:q0 + q_batch] = best_i.to(torch.int32)
        out_d[q0:q0 + q_batch] = best_d.to(torch.float32)
    return out_n, out_d


def separated_clusters(X: torch.Tensor, truth, kth_max: float) -> bool:
    """True if, for the clusters ``truth`` labels (contiguous id ranges), every
    point of another cluster is farther than kth_max from every point of its
    own: with m_c the fp64 mean and r_c the largest distance of a member to it,
    |x - y| >= |m_c - m_c'| - r_c - r_c' (triangle inequality).  Then the
    brute force over a query's own cluster is the brute force over all points."""
    import numpy as np
    t = np.asarray(truth)
    cuts = np.flatnonzero(t[1:] != t[:-1]) + 1
    b = np.concatenate([[0], cuts, [len(t)]])
    ms, rs = [], []
    for i in range(len(b) - 1):
        P = X[int(b[i]):int(b[i + 1])].double()
        m = P.mean(0)
        ms.append(m)
        rs.append(float(torch.sqrt(((P - m) ** 2).sum(1)).max()) * (1 + 1e-9))
    for i in range(len(ms)):
        for j in range(i + 1, len(ms)):
            if float(torch.linalg.norm(ms[i] - ms[j])) - rs[i] - rs[j] <= kth_max:
                return False
    return True
