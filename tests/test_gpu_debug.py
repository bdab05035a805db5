"""The debug build (lib/libkdb_dbg.so: a guard band after every workspace
array, filled before and verified after each kdb_mst / kdb_nmi call, and device
bounds checks on component ids in the hook, jump, merge and round kernels) over
small cases -- this pool's replacement for compute-sanitizer, which is closed
on it.  Each case also checks its result against the oracle
(tools/debug_cases.py); a guard or bounds violation surfaces as KDB_EINTERNAL.
"""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DBG = os.path.join(ROOT, "paper_2009_04552_b200", "lib", "libkdb_dbg.so")


@pytest.mark.parametrize("case", ["golden", "c1", "fallback", "edgecols", "inexact", "nmi", "poison", "c4slice"])
def test_debug_build_case(case):
    if not os.path.exists(DBG):
        subprocess.check_call(["make", "-C", ROOT, os.path.relpath(DBG, ROOT)])
    env = dict(os.environ, KDB_LIBRARY=DBG)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "debug_cases.py"), case], env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    assert f"case {case}: ok" in p.stdout


def test_poison_with_product_build():
    """The same workspace-poisoning and output-guard case on the product build."""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "debug_cases.py"), "poison"],
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
