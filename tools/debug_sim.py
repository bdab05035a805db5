import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2009_04552_b200 as kdb
from datagen import random_graph
from tests.kdb_harness import run_gpu, oracle_run
for seed in [7, 8, 9]:
  for sym in [False, True]:
    nbr, dist = random_graph(3000, 8, seed, levels=4, symmetric=sym, pad_frac=0.1, local=40)
    eps = np.float32(np.quantile(dist[np.isfinite(dist)].astype(np.float64), 0.6))
    exp = oracle_run(nbr, dist, 3, eps)
    E = set(zip(exp['msf_a'].tolist(), exp['msf_b'].tolist()))
    for P in [0, 1, 2, 3, 4, 5, 8]:
        got = run_gpu(nbr, dist, 3, eps, comm=kdb.Comm.sim(P) if P else None)
        G = set(zip(got['msf_a'].tolist(), got['msf_b'].tolist()))
        print(seed, sym, P, 'ok' if G == E else f'DIFF extra={sorted(G-E)[:4]} missing={sorted(E-G)[:4]}', got['stats']['rounds'])
