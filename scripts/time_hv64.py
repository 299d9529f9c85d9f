"""Calls the fp64 H.V (hv_f64) at a config's shape a few times (for ncu)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
s = int(sys.argv[2]) if len(sys.argv) > 2 else 65
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
q = datasets.CONFIGS[name]()
ctx = wg.Context(0)
ctx.set_data(q.X)
ctx.set_hyper([*q.lengthscales, q.signal, q.noise])
V = np.random.default_rng(0).standard_normal((q.X.shape[0], s))
for _ in range(reps):
    ctx.hv_f64(V)
print("ok")
