"""Seeded synthetic input generators for the kNN-DBSCAN clustering stage.

This package is shared by BOTH sides of the parity check (the CPU oracle in
``oracle/`` and the CUDA product path in ``paper_2009_04552_b200/``).  It holds
none of the method's arithmetic: it only produces inputs -- point sets, the
CPU brute-force k-NN graph of small point sets (the paper's input, PAPER.md:517
"the directed k-nearest neighbor graph G_k"), random graphs with adversarial
structure, and the epsilon rule of the configs.  It never imports either side.
Large graphs come from the package's kNN-graph builder (a separate, separately
timed input stage, paper_2009_04552_b200/knng.py; it
shares no code with the clustering kernels), which the callers (bench.py,
tests/) import directly.

Recipes follow BASELINE.json ``configs`` and SURVEY.md §8(d).
"""
from .points import (gen_c1, gen_c2, gen_c3, gen_c4, gen_c5, gen_config_points,
                     CONFIGS)
from .knn_cpu import knn_bruteforce, knn_rows_bruteforce
from .graphs import random_graph, eps_from_graph

__all__ = [
    "gen_c1", "gen_c2", "gen_c3", "gen_c4", "gen_c5", "gen_config_points",
    "CONFIGS", "knn_bruteforce", "knn_rows_bruteforce", "random_graph",
    "eps_from_graph",
]
