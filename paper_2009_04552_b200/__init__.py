"""B200-native kNN-DBSCAN clustering stage (arXiv 2009.04552).

The hot path is ``libkdb.so`` (hand-written sm_100a CUDA, C-ABI in
``include/kdb.h``); ``kdb`` is its thin ctypes binding.
"""
from .kdb import (Comm, Graph, KdbError, core_mark, kdbscan, kdbscan_sweep, label, launch_count, lib, mst, mst_inexact, nmi,
                  profile, profile_read, profile_reset, unpack_core, workspace_bytes, EXPORTS, LIB_PATH,
                  set_option, get_option, reset_options, option_names, options_from_env)

__all__ = ["Comm", "Graph", "KdbError", "core_mark", "kdbscan", "kdbscan_sweep", "label", "launch_count", "lib", "mst", "mst_inexact", "nmi",
           "profile", "profile_read", "profile_reset", "unpack_core", "workspace_bytes", "EXPORTS",
           "LIB_PATH", "set_option", "get_option", "reset_options", "option_names", "options_from_env"]
