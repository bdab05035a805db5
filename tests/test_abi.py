"""CPU-side checks of the C-ABI library (-m "not gpu"): it loads without a GPU,
exports every symbol include/kdb.h declares, and rejects invalid arguments
before launching anything (host-side validation, include/kdb.h conventions).
"""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kdb.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kdb_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import paper_2009_04552_b200 as kdb
    if not os.path.exists(kdb.LIB_PATH):
        subprocess.check_call(["make", "-C", ROOT, os.path.relpath(kdb.LIB_PATH, ROOT)])
    return kdb.lib()


def test_header_declares_the_three_calls():
    fns = declared_functions()
    for f in ("kdb_core_mark", "kdb_mst", "kdb_label", "kdb_mst_workspace_bytes"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    import paper_2009_04552_b200 as kdb
    fns = declared_functions()
    missing = [f for f in fns if not hasattr(lib, f)]
    assert not missing, missing
    assert sorted(kdb.EXPORTS) == fns
    # nm agrees (dynamic symbol table)
    out = subprocess.run(["nm", "-D", "--defined-only", kdb.LIB_PATH], capture_output=True, text=True).stdout
    for f in fns:
        assert re.search(rf"\bT {f}$", out, flags=re.M), f


def _graph(n_total=10, row_begin=0, n_rows=10, k=4, nbr=0x1000, dist=0x2000, flags=0, edge_cols=0):
    import paper_2009_04552_b200.kdb as K
    return K._Graph(n_total, row_begin, n_rows, k, nbr, dist, flags, edge_cols)


@pytest.mark.parametrize("kw,M,eps", [
    (dict(), 5, 0.5),                      # M > k
    (dict(), 0, 0.5),                      # M < 1
    (dict(), 2, 0.0),                      # eps not > 0
    (dict(), 2, float("inf")),             # eps not finite
    (dict(), 2, float("nan")),
    (dict(k=0), 1, 0.5),                   # k < 1
    (dict(n_rows=11), 2, 0.5),             # rows beyond n_total
    (dict(row_begin=-1), 2, 0.5),
    (dict(nbr=0), 2, 0.5),                 # NULL
    (dict(dist=0x2004), 2, 0.5),           # misaligned
    (dict(flags=8), 2, 0.5),               # unknown flag
    (dict(edge_cols=-1), 2, 0.5),          # edge_cols < 0
    (dict(edge_cols=5), 2, 0.5),           # edge_cols > k
])
def test_core_mark_validation(lib, kw, M, eps):
    g = _graph(**kw)
    rc = lib.kdb_core_mark(C.byref(g), M, eps, C.c_void_p(0x3000), None, None)
    assert rc == 1  # KDB_EINVAL, nothing launched
    assert lib.kdb_last_error()


def test_mst_validation_and_workspace(lib):
    g = _graph()
    assert lib.kdb_mst_workspace_bytes(C.byref(g), None) > 0
    exact = _graph(flags=1)
    # exact graphs need no in-edge lists
    assert lib.kdb_mst_workspace_bytes(C.byref(exact), None) < lib.kdb_mst_workspace_bytes(C.byref(g), None)
    cnt = C.c_int64(); tot = C.c_double()
    P = C.c_void_p
    # workspace too small -> ENOMEM before any launch
    rc = lib.kdb_mst(C.byref(g), 0.5, P(0x100), P(0x200), P(0x300), P(0x400), P(0x500), 9,
                     C.byref(cnt), C.byref(tot), P(0x1000), 16, None, None)
    assert rc == 2
    # NULL host outputs
    rc = lib.kdb_mst(C.byref(g), 0.5, P(0x100), P(0x200), P(0x300), P(0x400), P(0x500), 9,
                     None, None, P(0x1000), 1 << 40, None, None)
    assert rc == 1
    assert lib.kdb_status_string(2) == b"KDB_ENOMEM"


def test_edge_cols_workspace(lib):
    """edge_cols = k is the default; edge_cols < k needs no extra workspace (the
    kernels read the first edge_cols columns in place, kdb.h); the general-mode
    in-edge lists shrink with it."""
    ws = lambda **kw: lib.kdb_mst_workspace_bytes(C.byref(_graph(n_total=1000, n_rows=1000, k=32, **kw)), None)
    assert ws(edge_cols=32) == ws(edge_cols=0)
    assert ws(edge_cols=8) < ws(edge_cols=0)
    wx = lambda **kw: lib.kdb_mst_workspace_bytes(C.byref(_graph(n_total=1000, n_rows=1000, k=32, flags=1, **kw)), None)
    assert wx(edge_cols=8) <= wx(edge_cols=0)
    assert lib.kdb_mst_workspace_bytes(C.byref(_graph(edge_cols=9)), None) == 0  # invalid -> 0


def test_sim_comm_lifecycle(lib):
    h = C.c_void_p()
    assert lib.kdb_comm_create_sim(C.byref(h), 4) == 0 and h.value
    g = _graph(n_total=10, row_begin=2, n_rows=8)
    # sim needs the full graph
    assert lib.kdb_core_mark(C.byref(g), 2, 0.5, C.c_void_p(0x3000), h, None) == 1
    lib.kdb_comm_destroy(h)
    assert lib.kdb_comm_create_sim(C.byref(h), 0) == 1


def test_knng_library_exports_every_declared_symbol():
    """libknng.so (the kNN-graph builder stage, include/knng.h) loads without a
    GPU and exports every declared entry point."""
    from paper_2009_04552_b200 import knng
    if not os.path.exists(knng.LIB_PATH):
        subprocess.check_call(["make", "-C", ROOT, os.path.relpath(knng.LIB_PATH, ROOT)])
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "knng.h")).read(), flags=re.S)
    fns = sorted(set(re.findall(r"\b(knng_[a-z_0-9]+)\s*\(", src)))
    assert fns == ["knng_brute", "knng_exact_row", "knng_grid", "knng_grid_rows", "knng_grid_ws", "knng_ladder"]
    L = C.CDLL(knng.LIB_PATH)
    assert all(hasattr(L, f) for f in fns)
    out = subprocess.run(["nm", "-D", "--defined-only", knng.LIB_PATH], capture_output=True, text=True).stdout
    for f in fns:
        assert re.search(rf"\bT {f}$", out, flags=re.M), f
    # host-side argument checks, nothing launched (D out of range / k >= n)
    L.knng_brute.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 8
    assert L.knng_brute(None, 10, 65, 3, 8, *([None] * 8)) == 4
    assert L.knng_brute(None, 10, 3, 10, 16, *([None] * 8)) == 4


def test_mst_inexact_rejects_int32_overflowing_cut_counts(lib):
    """The cut entries of kdb_mst_inexact live in survivor buffers whose counts
    CUB takes as int: n_rows * edge_cols >= 2^31 - 1 is EINVAL before any launch."""
    P = C.c_void_p
    cnt = C.c_int64(); tot = C.c_double()
    n = (1 << 31) // 100 + 1          # n * k just above 2^31 - 1 with k = 100
    g = _graph(n_total=n, n_rows=n, k=100)
    rc = lib.kdb_mst_inexact(C.byref(g), C.c_float(0.5), P(0x100), 2, P(0x200), P(0x300), P(0x400), P(0x500), n - 1,
                             C.byref(cnt), C.byref(tot), P(0x1000), C.c_size_t(1 << 40), None)
    assert rc == 1 and b"2^31" in lib.kdb_last_error()
    g = _graph(n_total=n, n_rows=n, k=100, edge_cols=50)  # the bound is on edge_cols columns
    rc = lib.kdb_mst_inexact(C.byref(g), C.c_float(0.5), P(0x100), 2, P(0x200), P(0x300), P(0x400), P(0x500), n - 1,
                             C.byref(cnt), C.byref(tot), P(0x1000), C.c_size_t(16), None)
    assert rc == 2  # passes the guard, then the (tiny) workspace is too small: ENOMEM, nothing launched


def test_debug_build_exports_and_guards(lib):
    """lib/libkdb_dbg.so (guard bands + device bounds checks, tests/test_gpu_debug.py)
    exports the same C-ABI and asks for more workspace (its guard bands)."""
    import paper_2009_04552_b200 as kdb
    dbg = os.path.join(os.path.dirname(kdb.LIB_PATH), "libkdb_dbg.so")
    if not os.path.exists(dbg):
        subprocess.check_call(["make", "-C", ROOT, os.path.relpath(dbg, ROOT)])
    D = C.CDLL(dbg)
    assert all(hasattr(D, f) for f in declared_functions())
    D.kdb_mst_workspace_bytes.restype = C.c_size_t
    g = _graph(n_total=1000, n_rows=1000, k=32, flags=1)
    assert D.kdb_mst_workspace_bytes(C.byref(g), None) > lib.kdb_mst_workspace_bytes(C.byref(g), None)


def test_tuning_options_are_explicit_not_environment(lib, monkeypatch):
    """Tuning options come only from kdb_set_option (include/kdb.h): an unknown
    name is rejected, set/get/reset round-trip, and a KDB_* environment
    variable does not reach the library (the binding forwards it only when
    asked: options_from_env)."""
    import paper_2009_04552_b200 as kdb
    names = kdb.option_names()
    assert "KDB_LIGHT" in names and "KDB_FILTER" in names and len(names) == len(set(names))
    assert lib.kdb_set_option(b"KDB_NO_SUCH_OPTION", 1) == 1  # KDB_EINVAL
    assert lib.kdb_get_option(b"KDB_NO_SUCH_OPTION", None) == -1
    kdb.reset_options()
    monkeypatch.setenv("KDB_LIGHT", "3")
    assert kdb.get_option("KDB_LIGHT") is None  # the environment alone changes nothing
    assert kdb.options_from_env() == {"KDB_LIGHT": 3}
    assert kdb.get_option("KDB_LIGHT") == 3
    kdb.set_option("KDB_FILTER", 0)
    assert kdb.get_option("KDB_FILTER") == 0
    kdb.reset_options()
    assert all(kdb.get_option(n) is None for n in names)
    # no getenv of a tuning option is left in the library's sources
    csrc = os.path.join(ROOT, "paper_2009_04552_b200", "csrc")
    for f in os.listdir(csrc):
        src = open(os.path.join(csrc, f)).read()
        for n in names:
            assert f'getenv("{n}")' not in src, (f, n)
