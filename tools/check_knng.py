import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from datagen.knng_gpu import build_knng_grid
from datagen import knn_bruteforce, gen_c4
rng = np.random.default_rng(0)
for (n, d, k) in [(3000, 2, 16), (20000, 3, 100), (5000, 5, 30), (10000, 3, 7)]:
    X = rng.standard_normal((n, d)).astype(np.float32)
    X[rng.integers(0, n, n // 50)] = X[rng.integers(0, n, n // 50)]
    t = time.time(); nbr, dist, info = build_knng_grid(X, k); torch.cuda.synchronize()
    nb, db = knn_bruteforce(X, k)
    print(n, d, k, 'nbr eq', np.array_equal(nbr.cpu().numpy(), nb), 'dist eq', np.array_equal(dist.cpu().numpy(), db), info, f'{time.time()-t:.2f}s')
# C4 scaled sample check
X, _ = gen_c4(0, n_per=640_000)
t = time.time(); nbr, dist, info = build_knng_grid(X, 100); torch.cuda.synchronize(); print('C4/10 build', time.time()-t, info)
rows = rng.integers(0, len(X), 20)
from datagen.knn_cpu import knn_rows_bruteforce
nb, db = knn_rows_bruteforce(X, rows, 100)
print('C4/10 sampled rows eq', np.array_equal(nbr[rows].cpu().numpy(), nb), np.array_equal(dist[rows].cpu().numpy(), db))
