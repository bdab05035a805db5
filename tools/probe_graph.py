import sys, ctypes as C, torch, numpy as np
sys.path.insert(0, '.')
from datagen import gen_config_points
from datagen.knng_gpu import build_knng_grid
L = C.CDLL('./tools/probe_graph.so'); L.probe_gather.restype = C.c_float
L.probe_gather.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
X, _ = gen_config_points('C4', 0, 1.0)
nbr, dist, info = build_knng_grid(X, 100)
N = len(X)
names = ['nbr+gather', '-', '+dist', '+comp[v]', '+head r/w', '+min/atomic Kc (C=N/3)']
for comps in (N, N // 3, N // 50):
    comp = (torch.arange(N, dtype=torch.int64, device='cuda') * comps // N).to(torch.int32)
    Kc = torch.full((N,), -1, dtype=torch.int64, device='cuda')
    head = torch.zeros(N, dtype=torch.int16, device='cuda')
    for stride in (1, 5):
        for mode in (0, 2, 3, 4, 5):
            head.zero_()
            ms = L.probe_gather(nbr.data_ptr(), dist.data_ptr(), 100, 0, N, stride, comp.data_ptr(), mode, Kc.data_ptr(), head.data_ptr())
            print(f"comps {comps} stride {stride} mode {mode} {names[mode]:>24}: {ms:.2f} ms  {N//stride*100/ms/1e9:.3g} Tentries/s")
