"""H.V relative error of the three kernels on diagonal-dominant (config 1) and
dense-neighbourhood (config-3-like: d=3 uniform inputs, unit lengthscales) data."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

ctx = wg.Context(0)
cases = []
p = datasets.config1()
cases.append(("config1 n=13500 d=26", p.X, p.V, p.lengthscales, 1.0, 0.1, 256))
rng = np.random.default_rng(0)
X3 = rng.uniform(size=(20000, 3)).astype(np.float32)
V3 = rng.standard_normal((20000, 65)).astype(np.float32)
cases.append(("c3-like n=20000 d=3 ls=1", X3, V3, np.ones(3), 1.0, 0.5, 200))
X0 = datasets.config0().X
V0 = rng.standard_normal((2048, 17)).astype(np.float32)
cases.append(("config0 n=2048 d=8 ls=1", X0, V0, np.ones(8), 1.0, 0.5, 2048))
for name, X, V, ls, sf, sig, rows in cases:
    ctx.set_data(X)
    ctx.set_hyper([*ls, sf, sig])
    ref = orc.hv_rows(X, ls, sf, sig, V, 0, rows)
    for impl in ("simt", "tc"):
        ctx.set_hv_impl(impl)
        out = ctx.hv(V)[:rows]
        e = np.linalg.norm(out - ref) / np.linalg.norm(ref)
        print(f"{name:28s} {impl:8s} rel {e:.3e}")
