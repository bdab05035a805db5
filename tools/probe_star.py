import time, numpy as np, torch, paper_2009_04552_b200 as kdb
for n in (20000, 100000):
    k = 4
    nbr = np.zeros((n, k), np.int32); dist = np.zeros((n, k), np.float32)
    rng = np.random.default_rng(0)
    for v in range(n):
        others = rng.choice(n - 1, k - 1, replace=False) + 1
        others = others[others != v][: k - 1]
        while len(others) < k - 1: others = np.append(others, (v % (n - 1)) + 1)
        if v == 0:
            nbr[0] = np.arange(1, k + 1); dist[0] = 0.1
        else:
            nbr[v] = [0, *others]; dist[v] = [0.1, 0.5, 0.6, 0.7]
    g = kdb.Graph(torch.from_numpy(nbr).cuda(), torch.from_numpy(dist).cuda(), n_total=n)
    torch.cuda.synchronize(); t = time.time()
    bits, r, lab = kdb.kdbscan(g, 1, 1.0)
    torch.cuda.synchronize(); print(n, "edges", r.count, "time %.3f s" % (time.time() - t), "finalize_ms", r.stats["finalize_ms"])
