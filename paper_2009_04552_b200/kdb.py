"""Thin Python binding of libkdb.so (include/kdb.h) -- argument marshalling only.

Every step of the clustering stage runs in the CUDA kernels of
``csrc/kdb.cu``; this module passes ``tensor.data_ptr()`` and the current
torch stream through ctypes.  There is NO CPU fallback: if the shared library
is missing or fails to load, every call raises ``KdbError``.

Names follow the paper (Alg. 1): ``core_mark`` (lines 3-8),
``mst`` (ParallelLocalMST + DistributedCutMST, lines 10-12), ``label``
(ClusterBorder, line 13).
"""
from __future__ import annotations

import ctypes as C
import os
import dataclasses
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# KDB_LIBRARY: an alternative build of the same library (tuning experiments)
LIB_PATH = os.environ.get("KDB_LIBRARY") or os.path.join(_HERE, "lib", "libkdb.so")
KDB_GRAPH_EXACT = 1
KDB_GRAPH_REUSE = 2


class KdbError(RuntimeError):
    pass


_lib = None


class _Graph(C.Structure):
    _fields_ = [("n_total", C.c_int64), ("row_begin", C.c_int64), ("n_rows", C.c_int64),
                ("k_max", C.c_int32), ("nbr", C.c_void_p), ("dist", C.c_void_p),
                ("flags", C.c_uint32), ("edge_cols", C.c_int32)]


def lib():
    """Load libkdb.so (raises KdbError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise KdbError(f"libkdb.so not built ({LIB_PATH}); run `make` or __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P, i32, i64, f32, u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_uint32
    G = C.POINTER(_Graph)
    L.kdb_status_string.restype = C.c_char_p
    L.kdb_status_string.argtypes = [C.c_int]
    L.kdb_last_error.restype = C.c_char_p
    L.kdb_nccl_unique_id.argtypes = [P]
    L.kdb_comm_create_nccl.argtypes = [C.POINTER(P), P, C.c_int, C.c_int]
    L.kdb_comm_create_sim.argtypes = [C.POINTER(P), C.c_int]
    L.kdb_comm_destroy.argtypes = [P]
    L.kdb_comm_destroy.restype = None
    L.kdb_core_mark.argtypes = [G, i32, f32, P, P, P]
    L.kdb_nmi_workspace_bytes.argtypes = [i64]
    L.kdb_nmi_workspace_bytes.restype = C.c_size_t
    L.kdb_nmi.argtypes = [P, P, i64, C.POINTER(C.c_double), C.POINTER(i64), C.POINTER(i64), P, C.c_size_t, P]
    L.kdb_mst_inexact_workspace_bytes.argtypes = [G, i32]
    L.kdb_mst_inexact_workspace_bytes.restype = C.c_size_t
    L.kdb_mst_inexact.argtypes = [G, f32, P, i32, P, P, P, P, i64, C.POINTER(i64), C.POINTER(C.c_double), P,
                                  C.c_size_t, P]
    L.kdb_mst_workspace_bytes.argtypes = [G, P]
    L.kdb_mst_workspace_bytes.restype = C.c_size_t
    L.kdb_mst.argtypes = [G, f32, P, P, P, P, P, i64, C.POINTER(i64), C.POINTER(C.c_double), P,
                          C.c_size_t, P, P]
    L.kdb_label.argtypes = [G, f32, P, P, P, P]
    L.kdb_last_mst_stats.argtypes = [C.POINTER(C.c_double), C.c_int]
    L.kdb_profile_enable.argtypes = [C.c_int]
    L.kdb_profile_enable.restype = None
    L.kdb_profile_reset.restype = None
    L.kdb_launch_count.restype = C.c_longlong
    L.kdb_profile_read.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_double), C.POINTER(C.c_longlong), C.c_int]
    L.kdb_set_option.argtypes = [C.c_char_p, C.c_longlong]
    L.kdb_get_option.argtypes = [C.c_char_p, C.POINTER(C.c_longlong)]
    L.kdb_reset_options.restype = None
    L.kdb_option_name.argtypes = [C.c_int, C.POINTER(C.c_char_p)]
    _lib = L
    return L


# the symbols include/kdb.h declares (checked by the CPU test suite)
EXPORTS = sorted(["kdb_nccl_unique_id", "kdb_comm_create_nccl", "kdb_comm_create_sim", "kdb_comm_destroy",
                  "kdb_core_mark", "kdb_mst_workspace_bytes", "kdb_mst", "kdb_label", "kdb_last_mst_stats",
                  "kdb_profile_enable", "kdb_profile_reset", "kdb_launch_count", "kdb_profile_read",
                  "kdb_status_string", "kdb_last_error", "kdb_nmi_workspace_bytes", "kdb_nmi",
                  "kdb_mst_inexact_workspace_bytes", "kdb_mst_inexact", "kdb_set_option", "kdb_get_option",
                  "kdb_reset_options", "kdb_option_name"])


def option_names() -> list[str]:
    """The tuning options libkdb.so knows (include/kdb.h kdb_set_option)."""
    L, out, i = lib(), [], 0
    nm = C.c_char_p()
    while L.kdb_option_name(i, C.byref(nm)):
        out.append(nm.value.decode())
        i += 1
    return out


def set_option(name: str, value) -> None:
    """Override one tuning option process-wide (DESIGN.md §16 switches)."""
    _check(lib().kdb_set_option(name.encode(), int(value)), f"set_option({name})")


def get_option(name: str):
    """The caller-set value of an option, None if its default applies."""
    v = C.c_longlong()
    rc = lib().kdb_get_option(name.encode(), C.byref(v))
    if rc < 0:
        raise KdbError(f"unknown option {name}")
    return int(v.value) if rc == 1 else None


def reset_options() -> None:
    lib().kdb_reset_options()


def options_from_env(environ=None) -> dict:
    """Apply the KDB_* variables of `environ` that name options (bench.py and
    the tools scripts call this once at start; the library itself never reads
    the environment).  Returns what was applied."""
    environ = os.environ if environ is None else environ
    applied = {}
    for name in option_names():
        v = environ.get(name)
        if v not in (None, ""):
            set_option(name, int(v))
            applied[name] = int(v)
    return applied


def _check(rc: int, what: str):
    if rc != 0:
        L = lib()
        raise KdbError(f"{what}: {L.kdb_status_string(rc).decode()}: {L.kdb_last_error().decode()}")


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class Comm:
    """A kdb communicator: ``Comm.sim(P)`` (P virtual ranks on one GPU) or
    ``Comm.nccl(rank, nranks, group)`` (one rank per GPU; the 128-byte NCCL id
    is created on rank 0 and broadcast with torch.distributed)."""

    def __init__(self, handle, nranks: int, rank: int, kind: str):
        self.handle, self.nranks, self.rank, self.kind = handle, nranks, rank, kind

    @classmethod
    def sim(cls, nranks: int) -> "Comm":
        h = C.c_void_p()
        _check(lib().kdb_comm_create_sim(C.byref(h), int(nranks)), "kdb_comm_create_sim")
        return cls(h, nranks, 0, "sim")

    @classmethod
    def nccl(cls, rank: int, nranks: int, group=None) -> "Comm":
        from .dist import share_nccl_id

        def make_id():
            b = (C.c_ubyte * 128)()
            _check(lib().kdb_nccl_unique_id(C.cast(b, C.c_void_p)), "kdb_nccl_unique_id")
            return bytes(b)

        uid = share_nccl_id(rank, make_id, group)
        buf = (C.c_ubyte * 128)()
        C.memmove(buf, uid, 128)
        h = C.c_void_p()
        _check(lib().kdb_comm_create_nccl(C.byref(h), C.cast(buf, C.c_void_p), int(rank), int(nranks)),
               "kdb_comm_create_nccl")
        return cls(h, nranks, rank, "nccl")

    @classmethod
    def nccl_single(cls) -> "Comm":
        """A 1-rank NCCL communicator without torch.distributed (tests, bench
        --nccl1; with KDB_NCCL_FORCE=1 the library issues every collective)."""
        b = (C.c_ubyte * 128)()
        _check(lib().kdb_nccl_unique_id(C.cast(b, C.c_void_p)), "kdb_nccl_unique_id")
        h = C.c_void_p()
        _check(lib().kdb_comm_create_nccl(C.byref(h), C.cast(b, C.c_void_p), 0, 1), "kdb_comm_create_nccl")
        return cls(h, 1, 0, "nccl")

    def close(self):
        if self.handle is not None:
            lib().kdb_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class Graph:
    """This rank's rows of the kNN graph (device tensors, [n_rows, k]).

    edge_cols: candidate edges come from the first edge_cols columns of each
    row (0 = all k, reading #3; M = Def. 6's direct M-reachability)."""
    nbr: torch.Tensor
    dist: torch.Tensor
    n_total: int
    row_begin: int = 0
    exact: bool = False
    edge_cols: int = 0

    def __post_init__(self):
        if self.nbr.dtype != torch.int32 or self.dist.dtype != torch.float32:
            raise KdbError("nbr must be int32 and dist float32")
        if self.nbr.shape != self.dist.shape or self.nbr.dim() != 2:
            raise KdbError("nbr/dist must be [n_rows, k] tensors of equal shape")
        if not (self.nbr.is_cuda and self.dist.is_cuda):
            raise KdbError("nbr/dist must be CUDA tensors (there is no CPU path)")
        if not (self.nbr.is_contiguous() and self.dist.is_contiguous()):
            raise KdbError("nbr/dist must be contiguous")

    @property
    def k(self) -> int:
        return int(self.nbr.shape[1])

    @property
    def n_rows(self) -> int:
        return int(self.nbr.shape[0])

    def c(self) -> _Graph:
        return _Graph(int(self.n_total), int(self.row_begin), self.n_rows, self.k,
                      self.nbr.data_ptr(), self.dist.data_ptr(),
                      KDB_GRAPH_EXACT if self.exact else 0, int(self.edge_cols))


def _h(comm):
    return comm.handle if comm is not None else None


def core_mark(g: Graph, M: int, eps: float, comm: Comm | None = None, stream=None) -> torch.Tensor:
    """kdb_core_mark: int32[ceil(N/32)] bit words (uint32 semantics), replicated."""
    bits = torch.empty((g.n_total + 31) // 32, dtype=torch.int32, device=g.dist.device)
    gc = g.c()
    _check(lib().kdb_core_mark(C.byref(gc), int(M), float(eps), C.c_void_p(bits.data_ptr()),
                               _h(comm), _stream(stream)), "kdb_core_mark")
    return bits


def workspace_bytes(g: Graph, comm: Comm | None = None) -> int:
    gc = g.c()
    return int(lib().kdb_mst_workspace_bytes(C.byref(gc), _h(comm)))


class MstResult:
    def __init__(self, comp, a, b, w, count, weight, stats):
        self.comp, self.a, self.b, self.w = comp, a, b, w
        self.count, self.weight, self.stats = count, weight, stats


def mst(g: Graph, eps: float, core_bits: torch.Tensor, comm: Comm | None = None, stream=None,
        workspace: torch.Tensor | None = None, out: dict | None = None, reuse: bool = False) -> MstResult:
    """kdb_mst: exact MSF of the core-core candidate edges + component labels.
    reuse=True sets KDB_GRAPH_REUSE: the caller promises the same graph and
    workspace as the previous mst() call on that workspace (an eps sweep)."""
    dev = g.dist.device
    N = g.n_total
    o = out or {}
    comp = o.get("comp")
    if comp is None:
        comp = torch.empty(max(N, 1), dtype=torch.int32, device=dev)
    cap = max(N - 1, 0)
    a = o.get("a"); b = o.get("b"); w = o.get("w")
    if a is None:
        a = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        b = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        w = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
    nws = workspace_bytes(g, comm)
    if workspace is None or workspace.numel() < nws:
        workspace = torch.empty(max(nws, 256), dtype=torch.uint8, device=dev)
    cnt = C.c_int64(0)
    tot = C.c_double(0.0)
    gc = g.c()
    if reuse:
        gc.flags |= KDB_GRAPH_REUSE
    _check(lib().kdb_mst(C.byref(gc), float(eps), C.c_void_p(core_bits.data_ptr()),
                         C.c_void_p(comp.data_ptr()), C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                         C.c_void_p(w.data_ptr()), cap, C.byref(cnt), C.byref(tot),
                         C.c_void_p(workspace.data_ptr()), workspace.numel(), _h(comm), _stream(stream)),
           "kdb_mst")
    st = (C.c_double * 32)()
    lib().kdb_last_mst_stats(st, 32)
    stats = dict(rounds=int(st[0]), init_ms=st[1], min_edges_ms=st[2], contract_ms=st[3],
                 finalize_ms=st[4], inlist_ms=st[5], stall_rounds=int(st[6]), entries_read=int(st[7]),
                 filter_ms=st[8], heavy_ms=st[9], survivors=int(st[10]), heavy_rounds=int(st[11]),
                 tau=st[12], light_components=int(st[13]), fallback=int(st[14]),
                 filter_exceptions=int(st[15]), filter_slow_entries=int(st[16]),
                 payload_rows_bytes=st[17], payload_heavy_bytes=st[18], ell_reused=int(st[29]),
                 heavy_rank_ms=st[30], heavy_simred_ms=st[31])
    if st[19]:  # local-first contraction ran (multi-rank exact mode)
        stats["local_first"] = dict(local_ms_max=st[20], local_ms_sum=st[21], transition_ms=st[22],
                                    global_ms=st[23], global_components=int(st[24]), parked_rows=int(st[25]),
                                    transition_bytes=st[26], local_rounds=int(st[27]), global_scan_ms=st[28])
    m = cnt.value
    return MstResult(comp[:N], a[:m], b[:m], w[:m], m, tot.value, stats)


def mst_inexact(g: Graph, eps: float, core_bits: torch.Tensor, nparts: int, stream=None) -> MstResult:
    """kdb_mst_inexact: the paper's inexact MST over `nparts` contiguous groups
    (local MSFs + cut MSF over super vertices).  Same
    components as mst(); the forest is not the minimum one in general."""
    dev = g.dist.device
    N = g.n_total
    comp = torch.empty(max(N, 1), dtype=torch.int32, device=dev)
    cap = max(N - 1, 0)
    a = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    b = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    w = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
    gc = g.c()
    nws = int(lib().kdb_mst_inexact_workspace_bytes(C.byref(gc), int(nparts)))
    ws = torch.empty(max(nws, 256), dtype=torch.uint8, device=dev)
    cnt = C.c_int64(0)
    tot = C.c_double(0.0)
    _check(lib().kdb_mst_inexact(C.byref(gc), float(eps), C.c_void_p(core_bits.data_ptr()), int(nparts),
                                 C.c_void_p(comp.data_ptr()), C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                 C.c_void_p(w.data_ptr()), cap, C.byref(cnt), C.byref(tot),
                                 C.c_void_p(ws.data_ptr()), ws.numel(), _stream(stream)), "kdb_mst_inexact")
    st = (C.c_double * 20)()
    lib().kdb_last_mst_stats(st, 20)
    stats = dict(rounds=int(st[0]), cut_entries=int(st[10]), heavy_rounds=int(st[11]), local_components=int(st[13]),
                 local_ms=st[1] + st[2] + st[3] + st[5], cut_ms=st[8] + st[9],
                 payload_rows_bytes=st[17], payload_heavy_bytes=st[18])
    m = cnt.value
    return MstResult(comp[:N], a[:m], b[:m], w[:m], m, tot.value, stats)


def label(g: Graph, eps: float, core_bits: torch.Tensor, comp: torch.Tensor, stream=None,
          out: torch.Tensor | None = None) -> torch.Tensor:
    """kdb_label: canonical labels of this rank's rows (-1 = noise)."""
    labels = out if out is not None else torch.empty(max(g.n_rows, 1), dtype=torch.int32, device=g.dist.device)
    gc = g.c()
    _check(lib().kdb_label(C.byref(gc), float(eps), C.c_void_p(core_bits.data_ptr()),
                           C.c_void_p(comp.data_ptr()), C.c_void_p(labels.data_ptr()), _stream(stream)),
           "kdb_label")
    return labels[:g.n_rows]


def nmi(a: torch.Tensor, b: torch.Tensor, stream=None) -> tuple[float, int, int]:
    """kdb_nmi: (NMI, clusters in a, clusters in b) of two device int32 labellings
    (SPEC.md convention: NOISE = one pseudo-cluster; arithmetic-mean normalisation)."""
    if a.dtype != torch.int32 or b.dtype != torch.int32 or a.shape != b.shape or a.dim() != 1:
        raise KdbError("a, b must be 1-D int32 tensors of equal length")
    if not (a.is_cuda and b.is_cuda):
        raise KdbError("a, b must be CUDA tensors (there is no CPU path)")
    a = a.contiguous(); b = b.contiguous()
    n = int(a.numel())
    ws = torch.empty(max(int(lib().kdb_nmi_workspace_bytes(n)), 256), dtype=torch.uint8, device=a.device)
    v = C.c_double(0.0); ca = C.c_int64(0); cb = C.c_int64(0)
    _check(lib().kdb_nmi(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), n, C.byref(v), C.byref(ca),
                         C.byref(cb), C.c_void_p(ws.data_ptr()), ws.numel(), _stream(stream)), "kdb_nmi")
    return v.value, ca.value, cb.value


def profile(on: bool = True):
    """Enable/disable per-kernel event timing inside libkdb.so."""
    lib().kdb_profile_enable(1 if on else 0)


def profile_reset():
    lib().kdb_profile_reset()


def launch_count() -> int:
    return int(lib().kdb_launch_count())


def profile_read() -> dict:
    """{kernel name: (total device ms, launches)} since the last reset."""
    cap = 128
    names = C.create_string_buffer(16384)
    ms = (C.c_double * cap)()
    cnt = (C.c_longlong * cap)()
    n = lib().kdb_profile_read(names, 16384, ms, cnt, cap)
    nm = names.value.decode().split("\n")
    return {nm[i]: (ms[i], int(cnt[i])) for i in range(n)}


def kdbscan(g: Graph, M: int, eps: float, comm: Comm | None = None, stream=None, edge_cols: int | None = None,
            workspace: torch.Tensor | None = None, reuse: bool = False):
    """The whole clustering stage (Alg. 1): returns (core_bits, MstResult, labels).
    edge_cols overrides g.edge_cols (M = the paper's Def. 6 edge set)."""
    if edge_cols is not None:
        g = dataclasses.replace(g, edge_cols=int(edge_cols))
    bits = core_mark(g, M, eps, comm, stream)
    r = mst(g, eps, bits, comm, stream, workspace=workspace, reuse=reuse)
    lab = label(g, eps, bits, r.comp, stream)
    return bits, r, lab


def kdbscan_sweep(g: Graph, M: int, eps_values, comm: Comm | None = None, stream=None,
                  edge_cols: int | None = None):
    """Multi-eps sweep on ONE resident graph (Fig. eps_mnist protocol, PAPER.md:
    459-488: the kNN graph is built once and reused for every eps): one
    workspace, the three calls per eps.  Returns [(eps, core_bits, MstResult,
    labels)] in the order given."""
    if edge_cols is not None:
        g = dataclasses.replace(g, edge_cols=int(edge_cols))
    nws = workspace_bytes(g, comm)
    ws = torch.empty(max(nws, 256), dtype=torch.uint8, device=g.dist.device)
    out = []
    for i, eps in enumerate(eps_values):
        # after the first eps the graph and workspace are unchanged: the light
        # ELL built by the first call is reused (KDB_GRAPH_REUSE)
        bits, r, lab = kdbscan(g, M, eps, comm, stream, workspace=ws, reuse=i > 0)
        out.append((float(eps), bits, r, lab))
    return out


def unpack_core(bits: torch.Tensor, n: int) -> torch.Tensor:
    """uint8[n] core flags from the packed words (host-side helper for tests)."""
    b = bits.cpu().numpy().view("uint32")
    import numpy as np
    return torch.from_numpy(((b[np.arange(n) >> 5] >> (np.arange(n) & 31).astype(np.uint32)) & 1).astype(np.uint8))
