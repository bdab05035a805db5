"""Compatibility shim: the kNN-graph builder is a first-class stage of the
package now (paper_2009_04552_b200/knng.py, C-ABI include/knng.h)."""
from paper_2009_04552_b200.knng import build_knng_brute, build_knng_grid, estimate_radius  # noqa: F401
