"""One config-2 AP solve (5 epochs, blocks of 1000, engine from HV_IMPL) for a launch list."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

q = datasets.config2()
ctx = wg.Context(0, hv_impl=os.environ.get("HV_IMPL", "tc_f16"))
ctx.set_data(q.X)
ctx.set_hyper([*q.lengthscales, q.signal, q.noise])
rhs = np.random.default_rng(0).standard_normal((q.X.shape[0], 65)).astype(np.float32)
cfg = wg.SolverConfig(kind="ap", tol_mean=1e-12, tol_samples=1e-12, max_iterations=5, block_size=1000)
ctx.solve(rhs, cfg)
print("ok")
