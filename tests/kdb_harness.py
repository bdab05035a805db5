"""Shared helpers for the GPU parity tests: run the CUDA path through the C-ABI
binding and the oracle on the same seeded inputs, and compare element by element.
"""
from __future__ import annotations

import hashlib
import os

import numpy as np
import torch

import oracle
import paper_2009_04552_b200 as kdb


def kdb_opt(name: str, value) -> None:
    """Override a libkdb tuning option for the current test (tests/conftest.py
    resets every option after each test)."""
    kdb.set_option(name, int(value))


def run_gpu(nbr: np.ndarray, dist: np.ndarray, M: int, eps, *, exact: bool = False,
            comm: "kdb.Comm | None" = None, device: str = "cuda:0", edge_cols: int = 0):
    g = kdb.Graph(torch.from_numpy(np.ascontiguousarray(nbr, np.int32)).to(device),
                  torch.from_numpy(np.ascontiguousarray(dist, np.float32)).to(device),
                  n_total=nbr.shape[0], exact=exact, edge_cols=edge_cols)
    bits, r, lab = kdb.kdbscan(g, M, float(np.float32(eps)), comm=comm)
    torch.cuda.synchronize()
    return result_dict(bits, r, lab, nbr.shape[0])


def result_dict(bits, r, lab, n):
    return dict(core=kdb.unpack_core(bits, n).numpy(), comp=r.comp.cpu().numpy(),
                msf_a=r.a.cpu().numpy().astype(np.uint32), msf_b=r.b.cpu().numpy().astype(np.uint32),
                msf_w=r.w.cpu().numpy(), msf_weight=r.weight, labels=lab.cpu().numpy(), stats=r.stats)


def assert_parity(got: dict, exp: dict, rel_tol: float = 1e-6):
    """Bit-exact core flags, labels, MSF edge set and weights; fp64 total within
    rel_tol (north_star: 'MST total weight within 1e-6 relative')."""
    assert np.array_equal(got["core"], exp["core"]), "core flags differ"
    core = exp["core"].astype(bool)
    assert np.array_equal(got["comp"][core], exp["labels"][core]), "core component labels differ"
    assert np.all(got["comp"][~core] == -1), "non-core comp must be -1"
    assert np.array_equal(got["labels"], exp["labels"]), "labels differ"
    assert len(got["msf_a"]) == len(exp["msf_a"]), "MSF size differs"
    assert np.array_equal(got["msf_a"], exp["msf_a"]) and np.array_equal(got["msf_b"], exp["msf_b"]), \
        "MSF edge set differs"
    assert np.array_equal(got["msf_w"].view(np.uint32) & 0x7fffffff,
                          exp["msf_w"].view(np.uint32) & 0x7fffffff), "MSF weights differ"
    ew = exp["msf_weight"]
    assert abs(got["msf_weight"] - ew) <= rel_tol * max(abs(ew), 1e-300), \
        f"MSF weight {got['msf_weight']!r} vs {ew!r}"


def oracle_run(nbr, dist, M, eps, edge_cols=None):
    """The oracle's result, cached on disk by input hash for large inputs
    (a parity re-check need not re-run an oracle that takes
    minutes).  The cache holds only oracle/ outputs, keyed by a digest of the
    exact input bytes and parameters; $KDB_ORACLE_CACHE (default
    /tmp/kdb_oracle_cache; empty string: off).  Nothing depends on it being
    present -- a miss recomputes."""
    eps32 = np.float32(eps)
    cdir = os.environ.get("KDB_ORACLE_CACHE", "/tmp/kdb_oracle_cache")
    if not cdir or nbr.size < 2_000_000:
        return oracle.kdbscan(nbr, dist, M, eps32, edge_cols=edge_cols or None)
    h = hashlib.blake2b(digest_size=20)
    for a in (np.ascontiguousarray(nbr, np.int32), np.ascontiguousarray(dist, np.float32)):
        h.update(str(a.shape).encode())
        h.update(memoryview(a).cast("B"))
    h.update(f"M={M} eps={eps32.view(np.uint32)} ec={edge_cols or 0} v1".encode())
    path = os.path.join(cdir, h.hexdigest() + ".npz")
    if os.path.exists(path):
        try:
            with np.load(path) as z:
                out = {k: z[k] for k in z.files}
            out["msf_weight"] = float(out["msf_weight"])
            out["times"] = {"cached": path}
            return out
        except Exception:
            pass
    out = oracle.kdbscan(nbr, dist, M, eps32, edge_cols=edge_cols or None)
    try:
        os.makedirs(cdir, exist_ok=True)
        tmp = path + f".{os.getpid()}.tmp.npz"
        np.savez(tmp, **{k: np.asarray(v) for k, v in out.items() if k != "times"})
        os.replace(tmp, path)
    except OSError:
        pass
    return out
