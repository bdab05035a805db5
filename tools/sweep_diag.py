"""Per-eps statistics of a C4 eps sweep with the kept light ELL (diagnostic)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2009_04552_b200 as kdb
W = bench.make_workload("C4", 1.0, 0, "cuda:0")
g = kdb.Graph(W["nbr"], W["dist"], n_total=W["N"], exact=True)
eps_list = [float(np.float32(f * W["med"])) for f in (0.5, 1.0, 1.5, 2.0)]
for rep in range(2):
    out = kdb.kdbscan_sweep(g, W["M"], eps_list)
    torch.cuda.synchronize()
    for eps, bits, r, lab in out:
        s = r.stats
        print(json.dumps({"eps": eps, "reused": s["ell_reused"], "fallback": s["fallback"], "tau": s["tau"],
                          "survivors": s["survivors"], "light": s["light_components"],
                          "ms": {k: round(s[k], 2) for k in ("init_ms", "min_edges_ms", "filter_ms", "heavy_ms", "finalize_ms")}}))
