"""Short config-1 H.V run for ncu captures (a few launches on cuda:0)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

impl = sys.argv[1] if len(sys.argv) > 1 else "tc"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = datasets.config1()
ctx = wg.Context(0, hv_impl=impl)
ctx.set_data(p.X)
ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
for _ in range(reps):
    out = ctx.hv(p.V)
print("ok", impl, float(np.abs(out).sum()))
