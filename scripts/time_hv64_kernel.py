"""Calls the fp64 operator (hv_f64) at config 2's shape a few times with a
well-conditioned right-hand side, for kernel timing under ncu / ablation
builds (no solver: any operator output is fine).  usage: time_hv64_kernel.py [s]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 65
q = datasets.config2()
ctx = wg.Context(0)
ctx.set_data(q.X)
ctx.set_hyper([*q.lengthscales, q.signal, q.noise])
V = np.random.default_rng(0).standard_normal((q.X.shape[0], s))
for _ in range(4):
    ctx.hv_f64(V)
print("ok")
