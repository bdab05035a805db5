"""Diagnose C5 at 1/16 scale: timings, and rows whose lightest entry is missing from the MSF."""
import sys, time, os
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2009_04552_b200 as kdb
from datagen import CONFIGS, gen_config_points
from datagen.knng_gpu import build_knng_grid
from datagen.knn_cpu import knn_rows_bruteforce
cfg = CONFIGS['C5']
t = time.time(); X, _ = gen_config_points('C5', 0, 1/16); print('gen', time.time() - t, X.shape, flush=True)
t = time.time(); nbr, dist, info = build_knng_grid(X, 100); torch.cuda.synchronize(); print('build', time.time() - t, info, flush=True)
col = dist[:, 49].double(); n = col.numel()
med = float((torch.kthvalue(col, n // 2).values + torch.kthvalue(col, n // 2 + 1).values) / 2)
eps = float(np.float32(1.5 * med)); print('eps', eps)
g = kdb.Graph(nbr, dist, n_total=n, exact=True)
for it in range(2):
    t = time.time(); bits, r, lab = kdb.kdbscan(g, 50, eps); torch.cuda.synchronize(); print('kdbscan', time.time() - t, r.stats, flush=True)
core = (dist[:, 49] <= eps)
a = r.a.long(); b = r.b.long(); key = a * n + b
ids = torch.arange(n, device='cuda')
J0 = nbr[:, 0].long()
sel = core & (J0 >= 0) & (dist[:, 0] <= eps) & core[J0.clamp(min=0)]
v = ids[sel]; k0 = torch.minimum(v, J0[sel]) * n + torch.maximum(v, J0[sel])
pos = torch.searchsorted(key, k0).clamp(max=key.numel() - 1)
bad = (key[pos] != k0).nonzero().flatten()
print('rows missing their lightest edge:', bad.numel())
rows = v[bad[:5]].cpu().numpy()
for q in rows:
    print('row', q, 'nbr', nbr[q, :4].tolist(), 'dist', dist[q, :4].tolist(), 'comp', r.comp[q].item(), 'comp J0', r.comp[nbr[q,0]].item())
if len(rows):
    nb, db = knn_rows_bruteforce(X, rows, 100)
    print('graph rows exact:', np.array_equal(nbr[rows].cpu().numpy(), nb), np.array_equal(dist[rows].cpu().numpy(), db))
    for q in rows[:3]:
        m = (a == q) | (b == q)
        print('msf edges at', q, torch.stack([a[m], b[m]], 1).tolist()[:6], r.w[m].tolist()[:6])
os.environ['KDB_FILTER'] = '0'
t = time.time(); bits2, r2, lab2 = kdb.kdbscan(g, 50, eps); torch.cuda.synchronize(); print('nofilter', time.time() - t, r2.stats, flush=True)
print('same comp', torch.equal(r.comp, r2.comp), 'same msf', r.count == r2.count and torch.equal(r.a, r2.a) and torch.equal(r.b, r2.b))
