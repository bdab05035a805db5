#!/usr/bin/env python
"""Small invocations of the clustering stage for the DEBUG build
(lib/libkdb_dbg.so: workspace guard bands + device bounds checks, see
csrc/kdb_host.cuh Carver) -- the memory checks this pool's GPUs allow
(compute-sanitizer is closed on the pool: runs under it left GPUs needing a
reset).  Each case runs kdb_core_mark -> kdb_mst -> kdb_label through the C-ABI
and checks the result against the oracle, so a run that passes also produced
the right answer.  tests/test_gpu_debug.py runs every case with
KDB_LIBRARY=lib/libkdb_dbg.so.

  KDB_LIBRARY=paper_2009_04552_b200/lib/libkdb_dbg.so python tools/debug_cases.py <case>
cases: c1 (exact and general mode, sim ranks P=3), golden (W1-W3, every case),
c4slice (C4 recipe at 1e5 points, exact, the benchmarked knobs),
fallback (C1 with KDB_SURVCAP=0: the survivor overflow re-runs the rows phase),
edgecols (C1, edge_cols = M), inexact (C1, kdb_mst_inexact with 3 groups),
nmi (kdb_nmi on C1 labels), poison (C1 with the workspace pre-filled with
0x00 / 0xFF / 0xA5 and guard tails after every caller output buffer: identical
outputs, untouched tails -- an uninitialised-read and out-of-range-write check).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2009_04552_b200 as kdb  # noqa: E402
from datagen import CONFIGS, eps_from_graph, gen_c1, gen_config_points, knn_bruteforce  # noqa: E402
from tests.kdb_harness import assert_parity, oracle_run, run_gpu  # noqa: E402


def c1_graph():
    X, truth = gen_c1(0, n_per_blob=600, n_noise=120)
    nbr, dist = knn_bruteforce(X, 16)
    return nbr, dist, 8, float(eps_from_graph(dist, 8, 1.5)), truth


def case_c1():
    nbr, dist, M, eps, _ = c1_graph()
    exp = oracle_run(nbr, dist, M, eps)
    assert_parity(run_gpu(nbr, dist, M, eps, exact=True), exp)
    assert_parity(run_gpu(nbr, dist, M, eps, exact=False), exp)
    assert_parity(run_gpu(nbr, dist, M, eps, exact=True, comm=kdb.Comm.sim(3)), exp)


def case_golden():
    for f in ["w1_fig_cycle.json", "w2_fig_cut_mst.json", "w3_unit_square.json"]:
        g = json.load(open(os.path.join(ROOT, "tests", "golden", f)))
        sets = [(g["nbr"], g["dist"], g["cases"])]
        if "dup" in g:
            sets.append((g["dup"]["nbr"], g["dup"]["dist"], g["dup"]["cases"]))
        for nb, di, cases in sets:
            nb = np.array(nb, np.int32); di = np.array(di, np.float32)
            for c in cases:
                got = run_gpu(nb, di, c["M"], c["eps"], exact=False)
                assert got["labels"].tolist() == c["labels"], (f, c["case"])
                assert_parity(got, oracle_run(nb, di, c["M"], c["eps"]))


def case_c4slice():
    from paper_2009_04552_b200.knng import build_knng_grid
    X, _ = gen_config_points("C4", 0, 1e5 / 64e6)
    cfg = CONFIGS["C4"]
    nbr, dist, _ = build_knng_grid(X, cfg["k"])
    nb, di = nbr.cpu().numpy(), dist.cpu().numpy()
    M = cfg["M"]
    eps = float(np.float32(cfg["eps_factor"] * np.median(di[:, M - 1].astype(np.float64))))
    assert_parity(run_gpu(nb, di, M, eps, exact=True), oracle_run(nb, di, M, eps))


def case_fallback():
    kdb.set_option("KDB_SURVCAP", 0)
    kdb.set_option("KDB_LIGHT", 10)  # k = 16: the split runs only when asked for
    nbr, dist, M, eps, _ = c1_graph()
    got = run_gpu(nbr, dist, M, eps, exact=True)
    assert got["stats"]["fallback"] == 1
    assert_parity(got, oracle_run(nbr, dist, M, eps))


def case_edgecols():
    nbr, dist, M, eps, _ = c1_graph()
    assert_parity(run_gpu(nbr, dist, M, eps, exact=True, edge_cols=M), oracle_run(nbr, dist, M, eps, edge_cols=M))


def case_inexact():
    from oracle import inexact as oinx
    nbr, dist, M, eps, _ = c1_graph()
    g = kdb.Graph(torch.from_numpy(nbr).cuda(), torch.from_numpy(dist).cuda(), n_total=len(nbr))
    bits = kdb.core_mark(g, M, eps)
    r = kdb.mst_inexact(g, eps, bits, 3)
    exp = oinx.kdbscan_inexact(nbr, dist, M, np.float32(eps), 3)
    assert np.array_equal(r.a.cpu().numpy().astype(np.uint32), exp["msf_a"])
    assert np.array_equal(r.b.cpu().numpy().astype(np.uint32), exp["msf_b"])


def case_nmi():
    from oracle import nmi as onmi
    nbr, dist, M, eps, truth = c1_graph()
    got = run_gpu(nbr, dist, M, eps, exact=True)
    v, _, _ = kdb.nmi(torch.from_numpy(got["labels"]).cuda(), torch.from_numpy(truth).cuda())
    assert abs(v - onmi.nmi(got["labels"], truth)) <= 1e-9


def case_poison():
    nbr, dist, M, eps, _ = c1_graph()
    exp = oracle_run(nbr, dist, M, eps)
    N = len(nbr)
    g = kdb.Graph(torch.from_numpy(nbr).cuda(), torch.from_numpy(dist).cuda(), n_total=N, exact=True)
    ref = None
    T = 64  # guard tail elements after every caller output
    for fill in (0x00, 0xFF, 0xA5):
        ws = torch.full((kdb.workspace_bytes(g) + 4096,), fill, dtype=torch.uint8, device="cuda")
        out = {x: torch.full((N + T,), 0x7B7B7B7B, dtype=torch.int32, device="cuda") for x in ("comp", "a", "b")}
        out["w"] = torch.full((N + T,), -7.0, dtype=torch.float32, device="cuda")
        lab = torch.full((N + T,), 0x7B7B7B7B, dtype=torch.int32, device="cuda")
        bits = kdb.core_mark(g, M, eps)
        r = kdb.mst(g, eps, bits, workspace=ws, out=out)
        lb = kdb.label(g, eps, bits, r.comp, out=lab)
        torch.cuda.synchronize()
        assert bool((out["comp"][N:] == 0x7B7B7B7B).all()) and bool((lab[N:] == 0x7B7B7B7B).all())
        cap = N - 1
        assert bool((out["a"][cap:] == 0x7B7B7B7B).all()) and bool((out["b"][cap:] == 0x7B7B7B7B).all())
        assert bool((out["w"][cap:] == -7.0).all())
        got = dict(core=kdb.unpack_core(bits, N).numpy(), comp=r.comp.cpu().numpy(), labels=lb.cpu().numpy(),
                   msf_a=r.a.cpu().numpy().astype(np.uint32), msf_b=r.b.cpu().numpy().astype(np.uint32),
                   msf_w=r.w.cpu().numpy(), msf_weight=r.weight)
        assert_parity(got, exp)
        if ref is None:
            ref = got
        for key in ("core", "comp", "labels", "msf_a", "msf_b", "msf_w"):
            assert np.array_equal(got[key], ref[key]), (fill, key)


if __name__ == "__main__":
    name = sys.argv[1]
    globals()[f"case_{name}"]()
    torch.cuda.synchronize()
    print(f"case {name}: ok")
