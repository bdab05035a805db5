import sys, ctypes as C, torch
sys.path.insert(0, '.')
from datagen import gen_config_points
from datagen.knng_gpu import build_knng_grid
L = C.CDLL('./tools/probe_passA2.so'); L.probe.restype = C.c_float
L.probe.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int]
X, _ = gen_config_points('C4', 0, 1.0)
nbr, dist, info = build_knng_grid(X, 100); del dist; torch.cuda.empty_cache()
N = len(X)
comp = (torch.arange(N, dtype=torch.int64, device='cuda') // 300).to(torch.int32)
compact = torch.empty((N, 4), dtype=torch.int32, device='cuda')
for mode, nm in [(0, 'ids from rows (64-B atom per 16 B)'), (1, 'ids from compact coalesced copy'), (2, 'ids from L2-resident array, same-cluster')]:
    print(nm, '%.2f ms' % L.probe(nbr.data_ptr(), compact.data_ptr(), 100, N, comp.data_ptr(), mode))
