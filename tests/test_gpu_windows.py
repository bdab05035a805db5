"""Full-size oracle parity of the BENCHMARKED path on C4 (64M points) and on C5
at 1/4 scale (64M points, 5-D) by exact cluster windows (tests/window_check.py:
the ten clusters are closed sub-graphs, so the whole-workload oracle result is
the union of per-window oracle runs).

The GPU runs the whole graph once, exactly as bench.py's step does
(kdb_core_mark -> kdb_mst -> kdb_label, KDB_GRAPH_EXACT, default knobs: filter,
fast path, fused round 1, CAS offers).  Then, for EVERY window:
  * the window is closed (checked on the device),
  * its input checksum equals the one stored with the oracle's digest
    (tests/golden/window_oracle_*.json, written by tools/window_parity.py from
    oracle/ runs only -- the committed log is profiles/r02/window_parity_*.json),
  * the digest of the GPU output restricted to the window equals the oracle's;
and the totals (forest size, fp64 weight within 1e-6) match the sum over the
windows.  One C4 window is also recomputed by the oracle live and compared
element by element (core, labels, MSF edge set and weights).
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

import paper_2009_04552_b200 as kdb
from tests import window_check as wc

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _golden(name):
    return json.load(open(os.path.join(ROOT, "tests", "golden", f"window_oracle_{name}.json")))


def _run(config, scale, live_window=None, order="inertial"):
    import bench
    W = bench.make_workload(config, scale, 0, torch.device("cuda:0"), order=order)
    gold = _golden((config if scale == 1.0 else config + "q") + ("i" if order == "inertial" else ""))
    assert gold["N"] == W["N"] and gold["k"] == W["k"] and gold["M"] == W["M"]
    assert f"{np.float32(W['eps']).view(np.uint32):08x}" == gold["eps_bits"]
    N = W["N"]
    g = kdb.Graph(W["nbr"], W["dist"], n_total=N, exact=True)
    # KDB_* variables of the environment (tools/ A/B scripts: a knob's full-size parity); none by default
    knobs = kdb.options_from_env()
    if knobs:
        print("knobs:", knobs)
    bits, r, lab = kdb.kdbscan(g, W["M"], W["eps"])
    torch.cuda.synchronize()
    full = dict(core=kdb.unpack_core(bits, N).numpy(), comp=r.comp.cpu().numpy(), labels=lab.cpu().numpy(),
                msf_a=r.a.cpu().numpy().astype(np.uint32), msf_b=r.b.cpu().numpy().astype(np.uint32),
                msf_w=r.w.cpu().numpy())
    wins = wc.cluster_windows(W["truth"])
    assert len(wins) == len(gold["windows"]) == 10
    covered = 0
    for i, win in enumerate(wins):
        gw = gold["windows"][str(i)]
        if wc.is_range(win):
            assert (gw["s"], gw["e"]) == win
        assert gw.get("n", wc.win_size(win)) == wc.win_size(win)
        assert wc.window_closed(W["nbr"], win), f"window {i} not closed"
        assert wc.input_checksum(W["nbr"], W["dist"], win) == gw["input_checksum"], f"window {i}: input changed"
        got = wc.gpu_window(full, win)
        assert got["edges_inside"]
        covered += got["span"][1] - got["span"][0]
        assert len(got["msf_a"]) == gw["msf_edges"]
        assert wc.digest(got["core"], got["labels"], got["msf_a"], got["msf_b"], got["msf_w"]) == \
            gw["oracle_digest"], f"window {i} differs from the oracle"
        assert np.array_equal(got["comp"][got["core"] > 0], got["labels"][got["core"] > 0])
    assert covered == r.count == sum(w["msf_edges"] for w in gold["windows"].values())
    tot = sum(w["msf_weight"] for w in gold["windows"].values())
    assert abs(r.weight - tot) <= 1e-6 * tot
    if live_window is not None:  # the oracle itself, element by element, on one window
        win = wins[live_window]
        nw, dw = wc.window_graph_host(W["nbr"], W["dist"], win)
        del W
        exp = wc.run_oracle(nw, dw, gold["M"], float(np.float32(np.uint32(int(gold["eps_bits"], 16)).view(np.float32))))
        assert exp["digest"] == gold["windows"][str(live_window)]["oracle_digest"]
        assert wc.compare(wc.gpu_window(full, win), exp) == []


def test_c4_full_size_windows_match_oracle():
    _run("C4", 1.0, live_window=7)


def test_c5_quarter_scale_windows_match_oracle():
    _run("C5", 0.25)


def test_c4_full_size_windows_generation_order():
    """The same parity with the generator's cluster-major ids (windows are id ranges)."""
    _run("C4", 1.0, order="generation")
