import sys, ctypes as C, torch
sys.path.insert(0, '.')
from datagen import gen_config_points
from datagen.knng_gpu import build_knng_grid
L = C.CDLL('./tools/probe_passA.so'); L.probe_passA.restype = C.c_float
L.probe_passA.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int, C.c_int, C.c_int]
X, _ = gen_config_points('C4', 0, 1.0)
nbr, dist, info = build_knng_grid(X, 100)
N = len(X)
comp = (torch.arange(N, dtype=torch.int64, device='cuda') // 300).to(torch.int32)
for carve, win in [(0, 0), (64, 0), (64, 1), (96, 1)]:
    for mode, nm in [(0, 'plain'), (1, 'gather evict_last'), (2, 'stream evict_first'), (3, 'both')]:
        print(f'carve {carve} MB window {win} {nm:20s} %.2f ms' % L.probe_passA(nbr.data_ptr(), dist.data_ptr(), 100, N, comp.data_ptr(), mode, carve, win))
