"""Is the inertial order (datagen/partition.py) bitwise reproducible on the GPU?
Computes the C4 permutation three times in one process and prints whether they
agree (the window goldens key the permuted graph by an input checksum)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from datagen import gen_config_points  # noqa: E402
from datagen.partition import inertial_order  # noqa: E402

X, _ = gen_config_points(sys.argv[1] if len(sys.argv) > 1 else "C4", 0, 1.0)
ps = []
for _ in range(3):
    t = time.time()
    ps.append(inertial_order(X, device="cuda"))
    print(f"perm in {time.time() - t:.1f} s, digest {int(np.bitwise_xor.reduce(ps[-1] * 2654435761 % (1 << 61)))}")
print("identical:", all(np.array_equal(ps[0], p) for p in ps[1:]))
