"""The exact cluster-window decomposition behind the full-size C4 / C5 parity
(tests/window_check.py, tools/window_parity.py), checked on CPU (-m "not gpu").

On a small instance of the C4 / C5 recipe (10 unit spheres, centres >= 3 apart)
the oracle on the WHOLE graph equals the union of the oracle on each closed
cluster window with ids shifted back (core flags, labels, the MSF edge set and
weights; total weight within 1e-6), and the helpers that slice the GPU output
reproduce the whole-graph result window by window.  A window that is not
closed is detected.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from datagen import CONFIGS, gen_config_points, knn_bruteforce
from tests import window_check as wc


@pytest.mark.parametrize("name,scale,order", [("C4", 0.00015, "generation"), ("C5", 0.00004, "generation"),
                                              ("C4", 0.00015, "inertial")])
def test_whole_graph_oracle_is_union_of_windows(name, scale, order):
    X, truth = gen_config_points(name, 0, scale)
    if order == "inertial":  # clusters become id sets, not ranges
        from datagen.partition import inertial_order
        perm = inertial_order(X, device="cpu")
        X, truth = X[perm], truth[perm]
    k, M = 32, 16  # smaller rows keep the brute force quick; the argument does not depend on k
    nbr, dist = knn_bruteforce(X, k)
    eps = float(np.float32(CONFIGS[name]["eps_factor"] * np.median(dist[:, M - 1].astype(np.float64))))
    full = oracle.kdbscan(nbr, dist, M, np.float32(eps))
    res = dict(core=full["core"], comp=np.where(full["core"] > 0, full["labels"], -1).astype(np.int32),
               labels=full["labels"], msf_a=full["msf_a"], msf_b=full["msf_b"], msf_w=full["msf_w"])
    wins = wc.cluster_windows(truth)
    assert len(wins) == 10
    tn, td = torch.from_numpy(nbr), torch.from_numpy(dist)
    total, edges = 0.0, 0
    assert all(wc.is_range(w) for w in wins) == (order == "generation")
    for win in wins:
        assert wc.window_closed(tn, win)
        nw, dw = wc.window_graph_host(tn, td, win)
        assert nw.min() >= 0 and nw.max() < wc.win_size(win)
        r = wc.run_oracle(nw, dw, M, eps)
        got = wc.gpu_window(res, win)
        assert wc.compare(got, r) == []
        assert wc.digest(got["core"], got["labels"], got["msf_a"], got["msf_b"], got["msf_w"]) == r["digest"]
        total += r["msf_weight"]
        edges += len(r["msf_a"])
    assert edges == len(full["msf_a"])
    assert abs(total - full["msf_weight"]) <= 1e-6 * full["msf_weight"]


def test_window_helpers_detect_violations():
    X, truth = gen_config_points("C4", 0, 0.0001)
    nbr, dist = knn_bruteforce(X, 8)
    wins = wc.cluster_windows(truth)
    s, e = wins[3]
    tn = torch.from_numpy(nbr.copy())
    assert wc.window_closed(tn, s, e)
    tn[s + 5, 2] = e  # an entry leaving the window
    assert not wc.window_closed(tn, s, e)
    # the checksum sees a one-bit change of a weight and a swapped id
    td = torch.from_numpy(dist.copy())
    c0 = wc.input_checksum(torch.from_numpy(nbr), td, s, e)
    td2 = td.clone(); td2.view(torch.int32)[s + 1, 1] ^= 1
    assert wc.input_checksum(torch.from_numpy(nbr), td2, s, e) != c0
    n2 = nbr.copy(); n2[s + 1, [0, 1]] = n2[s + 1, [1, 0]]
    assert wc.input_checksum(torch.from_numpy(n2), td, s, e) != c0
    # a wrong label / MSF edge fails the comparison
    nw, dw = wc.window_graph_host(torch.from_numpy(nbr), td, s, e)
    r = wc.run_oracle(nw, dw, 4, float(np.float32(np.median(dist[:, 3]) * 1.5)))
    got = dict(core=r["core"].copy(), comp=np.where(r["core"] > 0, r["labels"], -1).astype(np.int32),
               labels=r["labels"].copy(), msf_a=r["msf_a"].copy(), msf_b=r["msf_b"].copy(), msf_w=r["msf_w"].copy(),
               msf_weight=r["msf_weight"], edges_inside=True)
    assert wc.compare(got, r) == []
    bad = dict(got, labels=got["labels"].copy()); bad["labels"][0] += 1
    assert "labels" in wc.compare(bad, r)
    if len(got["msf_b"]):
        bad = dict(got, msf_b=got["msf_b"].copy()); bad["msf_b"][-1] ^= 1
        assert "msf edge set" in wc.compare(bad, r)
