import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libkdb.so")


import pytest


@pytest.fixture(autouse=True)
def _kdb_options_reset():
    """Every test starts and ends with libkdb's tuning options at their
    defaults (tests override them with kdb_harness.kdb_opt)."""
    yield
    mod = sys.modules.get("paper_2009_04552_b200.kdb")
    if mod is not None and mod._lib is not None:
        mod.reset_options()
