"""Point order by recursive inertial bisection -- input preparation, not the method.

PAPER.md:45: "Each MPI process loads a random N/p portion of the dataset.
Further, we partition the datasets using a standard inertial graph partitioning
algorithm to reduce the size of the edge cut."  The clustering stage receives
its points (and so the ids of the kNN graph) in that partitioned order: rank r
owns a contiguous id range, and with the partition applied the
range is a spatially compact piece of the data set.

Standard inertial bisection: a segment of points is split at the median of its
projections onto its principal axis of inertia (the eigenvector of the largest
eigenvalue of the segment's covariance), both halves recursively, until every
segment holds at most ``leaf`` points.  The recursion is carried to small
leaves (not only to p parts), so the order is also a locality order inside a
rank.  Ties in the projection keep the incoming order (stable sorts); all
statistics are fp64 prefix sums, so the permutation is deterministic for a
given input and device.

This module holds none of the clustering arithmetic; both sides of the parity
check receive the same permuted points and graph.
"""
from __future__ import annotations

import numpy as np


def _seg_sums(v, starts, ends):
    """Per-segment sums of v (fp64 [c, n], rows contiguous) over [starts, ends)
    via a prefix sum along the contiguous dimension -> [c, n_seg]."""
    import torch
    out = []
    for row in v:  # 1-D prefix sums (a device-wide scan; row-wise 2-D scans are far slower)
        cs = torch.cumsum(row, dim=0)
        cs = torch.cat([torch.zeros_like(cs[:1]), cs])
        out.append(cs[ends] - cs[starts])
    return torch.stack(out)


def _principal_axis(cov, iters: int = 40):
    """Dominant eigenvector of each symmetric PSD [d, d] matrix by power
    iteration from a fixed start (batched; batched eigh solvers reject the
    millions of tiny matrices of the deep levels).  A degenerate top eigenspace
    (an isotropic segment) yields some unit vector in it -- any such axis is an
    inertial axis."""
    import torch
    b, d, _ = cov.shape
    v = torch.linspace(1.0, 0.5, d, dtype=torch.float64, device=cov.device).expand(b, d).contiguous()
    for _ in range(iters):
        v = torch.bmm(cov, v[:, :, None])[:, :, 0]
        nrm = v.norm(dim=1, keepdim=True)
        v = torch.where(nrm > 0, v / torch.where(nrm > 0, nrm, torch.ones_like(nrm)), v)
    return v


def inertial_order(X, leaf: int = 64, device: str = "cuda", align: int = 1024):
    """Permutation (int64 numpy [n]) that lists the points of X (float32 [n, d])
    in recursive inertial-bisection order; X[perm] is the partitioned data set.
    Segments larger than two ``align``-id blocks are split at a block boundary
    nearest below the median (the clustering stage's tile round takes 1,024
    consecutive rows per tile: each tile is then one bisection piece)."""
    import torch
    Xt = torch.as_tensor(np.ascontiguousarray(X, np.float32) if isinstance(X, np.ndarray) else X)
    Xt = Xt.to(device=device)
    n, d = Xt.shape
    perm = torch.arange(n, device=device, dtype=torch.int64)
    starts = torch.zeros(1, dtype=torch.int64, device=device)
    ends = torch.full((1,), n, dtype=torch.int64, device=device)
    pos = torch.arange(n, device=device, dtype=torch.int64)
    iu = torch.triu_indices(d, d, device=device)
    while n > leaf and int((ends - starts).max()) > leaf:
        seg = torch.searchsorted(starts, pos, right=True) - 1          # segment of each position
        cnt = (ends - starts).to(torch.float64)
        x = Xt[perm].to(torch.float64).T.contiguous()                  # [d, n]
        mean = _seg_sums(x, starts, ends) / cnt[None, :]                # [d, n_seg]
        y = x - mean[:, seg]
        del x
        prod = y[iu[0]] * y[iu[1]]                                      # upper triangle of y y^T, [d(d+1)/2, n]
        cov_u = _seg_sums(prod, starts, ends).T                         # [n_seg, d(d+1)/2]
        del prod
        cov = torch.zeros(len(starts), d, d, dtype=torch.float64, device=device)
        cov[:, iu[0], iu[1]] = cov_u
        cov[:, iu[1], iu[0]] = cov_u
        axis = _principal_axis(cov)
        # deterministic sign: largest-magnitude component positive
        sgn = torch.sign(torch.gather(axis, 1, axis.abs().argmax(1, keepdim=True)))
        axis = axis * torch.where(sgn == 0, torch.ones_like(sgn), sgn)
        proj = (y * axis[seg].T).sum(0)
        del y
        # order inside each segment by projection (stable), segments stay in place
        o1 = torch.sort(proj, stable=True).indices
        o2 = torch.sort(seg[o1], stable=True).indices
        order = o1[o2]
        perm = perm[order]
        del proj, o1, o2, order, seg
        # split at the median; segments of >= 2 aligned blocks split at a block
        # boundary (block = ``align`` ids), so the pieces of ``align`` points
        # are exactly the id blocks a consumer tiles by
        q = (ends - starts) // align
        mid = torch.where(q >= 2, starts + (q // 2) * align, starts + (ends - starts) // 2)
        split = (ends - starts) > leaf
        new_s = torch.stack([starts, torch.where(split, mid, ends)], 1).reshape(-1)
        new_e = torch.stack([torch.where(split, mid, ends), ends], 1).reshape(-1)
        keep = new_e > new_s
        starts, ends = new_s[keep].contiguous(), new_e[keep].contiguous()
    return perm.cpu().numpy()
