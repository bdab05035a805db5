import sys, ctypes as C, torch, numpy as np
sys.path.insert(0, '.')
import bench
import paper_2009_04552_b200 as kdb
L = C.CDLL('./tools/probe_graph.so'); L.probe_gather.restype = C.c_float
L.probe_gather.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
W = bench.make_workload('C4', 1.0, 0, 'cuda:0')
N = W['N']
g = kdb.Graph(W['nbr'], W['dist'], n_total=N, exact=True)
ws = torch.empty(kdb.workspace_bytes(g), dtype=torch.uint8, device='cuda')
outs = {"comp": torch.empty(N, dtype=torch.int32, device='cuda'), "a": torch.empty(N, dtype=torch.int32, device='cuda'),
        "b": torch.empty(N, dtype=torch.int32, device='cuda'), "w": torch.empty(N, dtype=torch.float32, device='cuda')}
Kc = torch.full((N,), -1, dtype=torch.int64, device='cuda'); head = torch.zeros(N, dtype=torch.int16, device='cuda')
comp_fresh = (torch.arange(N, dtype=torch.int64, device='cuda') // 3).to(torch.int32)
def probe(tag, comp):
    ms = L.probe_gather(W['nbr'].data_ptr(), W['dist'].data_ptr(), 100, 0, N, 5, comp.data_ptr(), 3, Kc.data_ptr(), head.data_ptr())
    print(f'{tag}: {ms:.2f} ms')
probe('before kdb, fresh comp', comp_fresh)
probe('before kdb, outs comp (uninit)', outs['comp'])
bits = kdb.core_mark(g, W['M'], W['eps'])
r = kdb.mst(g, W['eps'], bits, workspace=ws, out=outs)
torch.cuda.synchronize()
print('kdb stats', r.stats)
probe('after kdb, fresh comp', comp_fresh)
probe('after kdb, outs comp (final labels)', outs['comp'])
