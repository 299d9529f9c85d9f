"""Accuracy of one library build's fp32 tc H.V (dev A/B companion): config 1
row sample and a dense config-3-like case against the fp64 oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

ctx = wg.Context(0)
out = []
for name, p in (("c1", datasets.config1()), ("c3like", datasets.config3(n=20000))):
    n = p.X.shape[0]
    V = p.V if p.V is not None else np.random.default_rng(3).standard_normal((n, 65)).astype(np.float32)
    ctx.set_data(p.X)
    ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
    o = ctx.hv(V)
    ref = orc.hv_rows(p.X, p.lengthscales, p.signal, p.noise, V, 0, 512)
    out.append(f"{name} rel {np.linalg.norm(o[:512] - ref) / np.linalg.norm(ref):.2e}")
print(" | ".join(out))
